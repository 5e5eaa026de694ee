#!/bin/bash
# Round evidence: GPU parity, smoke, bench lines (default c3, c2, c4, c4k, c5, alpha = 0 for c3 / c5,
# c4h / c3h (hierarchical index), c3q (Quest min/max), c1, reference), the ncu launch list of one timed step of the default command and ncu --set full
# captures.  usage: tools/gpu_round.sh <tag>
tag=${1:-r02}; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/${tag}_box.txt; nproc >> gpurun_out/${tag}_box.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc $?"
b() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/${tag}_bench_$name.json 2> gpurun_out/${tag}_bench_$name.err; echo -n "$name rc $? "; python tools/line_summary.py gpurun_out/${tag}_bench_$name.json; }
b default
b c2 --config c2
b c4 --config c4
b c4k --config c4k --no-cpu-baseline
b c5 --config c5 --no-cpu-baseline
b c3_alpha0 --config c3 --alpha 0 --no-cpu-baseline
b c5_alpha0 --config c5 --alpha 0 --no-cpu-baseline
b c4h --config c4h --no-cpu-baseline
b c3h --config c3h --no-cpu-baseline
b c3q --config c3q --no-cpu-baseline
b c1 --config c1 --no-cpu-baseline
b reference --impl reference --steps 5 --warmup 3
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,syslts__d_sectors_fill_sysmem.sum"
K="regex:score_kernel|rank_kernel|select_kernel|attn_kernel|cand_kernel|resolve_kernel|gather_kernel"
# default command (c3, 32 fill steps: steady-state misses): skip fill (32 x 32 layers x 16 chains x 3) + 3 warm-up graph steps (x 1536),
# then log one timed step (1536 launches: score, select, attention per layer and chain)
timeout 1500 /usr/local/cuda/bin/ncu --metrics $M --clock-control none -k "$K" -s $((32*1536 + 3*1536)) -c 1536 --csv \
  --log-file gpurun_out/${tag}_launches_default.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-isolated > gpurun_out/${tag}_ncu_default.out 2>&1
echo "launch list rc $?"; python tools/ncu_summary.py gpurun_out/${tag}_launches_default.csv > gpurun_out/${tag}_launches_default_summary.txt; cat gpurun_out/${tag}_launches_default_summary.txt
timeout 900 /usr/local/cuda/bin/ncu --metrics $M --clock-control none -k "$K" -s $((4*1536)) -c 1536 --csv \
  --log-file gpurun_out/${tag}_launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-isolated > gpurun_out/${tag}_ncu_c2.out 2>&1
echo "launch list c2 rc $?"; python tools/ncu_summary.py gpurun_out/${tag}_launches_c2.csv > gpurun_out/${tag}_launches_c2_summary.txt; cat gpurun_out/${tag}_launches_c2_summary.txt
# --set full: whole-batch launches (eager, chains = 1, same kernels as the graph) of c2, c3, c4 after
# 32 fill steps of 2 layers (6 launches per step): the first warm-up step's 2 x (score, select, attention)
for c in c2 c3 c4; do
  timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k "$K" -s $((32*6)) -c 6 -o gpurun_out/${tag}_full_$c -f \
    python bench.py --config $c --layers 2 --chains 1 --no-graph --fill 32 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-isolated > gpurun_out/${tag}_full_$c.out 2>&1
  echo "full $c rc $?"
  python tools/ncu_details.py gpurun_out/${tag}_full_$c.ncu-rep > gpurun_out/${tag}_full_$c.txt 2>&1
done
python tools/ncu_traffic.py ${tag} c2=gpurun_out/${tag}_full_c2.ncu-rep:64 c3=gpurun_out/${tag}_full_c3.ncu-rep:128 c4=gpurun_out/${tag}_full_c4.ncu-rep:16 \
  --link c3=gpurun_out/${tag}_launches_default.csv:8 > gpurun_out/${tag}_traffic.log 2>&1; cp profiles/${tag}_ncu_traffic.json gpurun_out/ 2>/dev/null
