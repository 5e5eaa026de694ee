#!/bin/bash
# ncu --set full of the select kernel (whole-batch launches, eager): per-source-line stall samples.
# usage: tools/gpu_ncu_sel.sh <tag> [configs...]
tag=${1:-ns}; shift; cfgs=${@:-c3}; mkdir -p gpurun_out
for c in $cfgs; do
  timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"rank_kernel|score_kernel" -s 64 -c 4 \
    -o gpurun_out/${tag}_sel_$c -f python bench.py --config $c --layers 2 --chains 1 --no-graph --fill 32 --steps 1 --warmup 1 \
    --no-e2e --no-cpu-baseline --no-isolated > gpurun_out/${tag}_sel_$c.out 2>&1
  echo "ncu $c rc $?"
done
