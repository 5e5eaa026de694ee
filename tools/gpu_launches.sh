#!/bin/bash
# per-kernel device times (ncu launch list, serialised, cold-ish) for c2/c3/c4 at 4 layers, no graph.
# usage: tools/gpu_launches.sh <tag> [configs...]
tag=${1:-ll}; shift; cfgs=${@:-c2 c3 c4}
mkdir -p gpurun_out
K='regex:score_kernel|topk_kernel|resolve_kernel|gather_kernel|attn_kernel|merge_kernel'
for c in $cfgs; do
  timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" --csv \
    --log-file gpurun_out/${tag}_launches_$c.csv python bench.py --config $c --layers 4 --chains 1 --no-graph --fill 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_ncu_$c.out 2>&1
  echo "== $c rc $?"
  python tools/ncu_summary.py gpurun_out/${tag}_launches_$c.csv
done
