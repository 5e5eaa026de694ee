#!/bin/bash
# round artefacts: default bench line (c3), c2 line, reference arm, launch list of the default command,
# ncu --set full of the step kernels.  usage: tools/gpu_round.sh <tag>
tag=${1:-r01}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${tag}_bench_default.json 2> gpurun_out/${tag}_bench_default.err; echo "default rc $?"
timeout 600 python bench.py --config c2 > gpurun_out/${tag}_bench_c2.json 2> gpurun_out/${tag}_bench_c2.err; echo "c2 rc $?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${tag}_bench_reference.json 2> gpurun_out/${tag}_bench_reference.err; echo "ref rc $?"
K="regex:select_kernel|resolve_kernel|gather_kernel|attn_kernel"
# default c3 command: fill 32 steps eager (32 layers x 16 chains x 4 kernels = 2048 per step) -> skip fill, log 2 graph steps
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" \
  -s $((32*2048)) -c 4096 --csv --log-file gpurun_out/${tag}_launches_default.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_ncu_default.out 2>&1
echo "launch list rc $?"
python tools/ncu_summary.py gpurun_out/${tag}_launches_default.csv
bash tools/gpu_full.sh ${tag}_full_c3 c3 "select_kernel|resolve_kernel|gather_kernel|attn_kernel" 256 4 2
for f in gpurun_out/${tag}_bench_default.json gpurun_out/${tag}_bench_c2.json gpurun_out/${tag}_bench_reference.json; do tail -1 $f | cut -c1-400; done
