#!/bin/bash
KVD_ATTN_TRACE=1 timeout 300 python bench.py --config c2 --layers 2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --chains 1 --no-graph 2>&1 >/dev/null | grep "attn trace" | tail -14
