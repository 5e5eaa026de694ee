#!/bin/bash
# per-kernel device times from an ncu launch list (gpu__time_duration + dram bytes), 4-layer copies.
# usage: tools/gpu_prof.sh <tag> [configs...]
tag=${1:-p}; shift
cfgs=${@:-c2 c3}
mkdir -p gpurun_out
K="regex:score_kernel|topk_kernel|resolve_kernel|gather_kernel|attn_kernel"
for c in $cfgs; do
  if [ $c = c2 ]; then skip=12; else skip=$((4*4*32)); fi
  timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" -s $skip -c 60 --csv \
    --log-file gpurun_out/${tag}_launches_$c.csv python bench.py --config $c --layers 4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_ncu_$c.out 2>&1
  echo "== $c rc $?"
  python tools/ncu_summary.py gpurun_out/${tag}_launches_$c.csv
done
