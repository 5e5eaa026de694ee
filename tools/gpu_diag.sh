#!/bin/bash
# phase traces of select / attention + c2 chain sweep.  usage: tools/gpu_diag.sh <tag>
tag=${1:-diag}; mkdir -p gpurun_out
for c in c2 c3 c4; do
  echo "== sel trace $c"
  KVD_TOPK_TRACE=1 timeout 300 python bench.py --config $c --layers 2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --chains 1 --no-graph --fill 4 2>&1 >/dev/null | grep "topk trace" | tail -9
  echo "== attn trace $c"
  KVD_ATTN_TRACE=1 timeout 300 python bench.py --config $c --layers 2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --chains 1 --no-graph --fill 4 2>&1 >/dev/null | grep "attn trace" | tail -7
done
for ch in 2 4 8; do
  timeout 300 python bench.py --config c2 --chains $ch --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_c2_ch$ch.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/${tag}_c2_ch$ch.json').read().strip().splitlines()[-1]);print('c2 chains $ch', round(d['value']), d['ms_per_step'])"
done
