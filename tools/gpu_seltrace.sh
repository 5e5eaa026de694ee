#!/bin/bash
for c in c2 c3; do
KVD_TOPK_TRACE=1 timeout 300 python bench.py --config $c --layers 2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --chains 1 --no-graph --fill 4 2>&1 >/dev/null | grep "topk trace" | tail -9
done
