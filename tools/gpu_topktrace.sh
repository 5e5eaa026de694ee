#!/bin/bash
for c in c2 c3 c4; do
echo "== $c"
KVD_TOPK_TRACE=1 timeout 300 python bench.py --config $c --layers 2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --chains 1 --no-graph --fill 1 2>&1 >/dev/null | grep "topk trace" | tail -7
done
