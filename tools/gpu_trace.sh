#!/bin/bash
# experiments build + phase traces (select / attention CTAs and warps).  usage: tools/gpu_trace.sh <tag> [cfg:chain ...]
tag=${1:-tr}; shift; specs=${@:-c2:0 c2:1 c3:0 c4:0}; mkdir -p gpurun_out
KVD_BUILD_EXPERIMENTS=1 python -c "from paper_2605_18071_b200 import build as b; b.build(force=True)" || exit 1
for sp in $specs; do c=${sp%%:*}; n=${sp##*:}
  echo "=== $c chain-size $n"; timeout 600 python tools/exp_trace.py --config $c --chain-size $n --reps 2 2>&1 | tail -16
done
