#!/bin/bash
# round artefacts: GPU parity, smoke, bench lines (default c3 / c2 / c4 / c5 / reference), the ncu
# launch list of the default command and ncu --set full captures.  usage: tools/gpu_round.sh <tag>
tag=${1:-r01}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc $?"
timeout 900 python bench.py > gpurun_out/${tag}_bench_default.json 2> gpurun_out/${tag}_bench_default.err; echo "default rc $?"
timeout 600 python bench.py --config c2 > gpurun_out/${tag}_bench_c2.json 2> gpurun_out/${tag}_bench_c2.err; echo "c2 rc $?"
timeout 900 python bench.py --config c4 > gpurun_out/${tag}_bench_c4.json 2> gpurun_out/${tag}_bench_c4.err; echo "c4 rc $?"
timeout 900 python bench.py --config c5 --no-cpu-baseline > gpurun_out/${tag}_bench_c5.json 2> gpurun_out/${tag}_bench_c5.err; echo "c5 rc $?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${tag}_bench_reference.json 2> gpurun_out/${tag}_bench_reference.err; echo "ref rc $?"
K="regex:score_kernel|topk_kernel|resolve_kernel|gather_kernel|attn_kernel|merge_kernel"
# default command (c3): 32 eager fill steps x 32 layers x 4 launches, 3 warm-up graph steps x 2048,
# then 2 timed graph steps (2048 launches each) are the ones logged
timeout 1200 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" \
  -s $((32*128 + 3*2048)) -c 4096 --csv --log-file gpurun_out/${tag}_launches_default.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_ncu_default.out 2>&1
echo "launch list rc $?"
python tools/ncu_summary.py gpurun_out/${tag}_launches_default.csv > gpurun_out/${tag}_launches_default_summary.txt; cat gpurun_out/${tag}_launches_default_summary.txt
# c2 (resident): 1 eager fill step (128 launches), 3 warm-up graph steps x 128, log 2 steps
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" \
  -s $((128 + 3*128)) -c 256 --csv --log-file gpurun_out/${tag}_launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_ncu_c2.out 2>&1
echo "launch list c2 rc $?"
python tools/ncu_summary.py gpurun_out/${tag}_launches_c2.csv > gpurun_out/${tag}_launches_c2_summary.txt; cat gpurun_out/${tag}_launches_c2_summary.txt
# --set full of one layer's kernels: c3 whole batch, unchained eager steps (2 layers, fill 4)
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k "$K" -s 32 -c 8 -o gpurun_out/${tag}_full_c3 -f \
  python bench.py --config c3 --layers 2 --chains 1 --no-graph --fill 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_full_c3.out 2>&1
echo "full c3 rc $?"
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k "$K" -s 8 -c 8 -o gpurun_out/${tag}_full_c2 -f \
  python bench.py --config c2 --layers 2 --chains 1 --no-graph --fill 1 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_full_c2.out 2>&1
echo "full c2 rc $?"
for f in gpurun_out/${tag}_bench_*.json; do echo $f; tail -1 $f | cut -c1-200; done
