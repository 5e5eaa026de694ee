#!/bin/bash
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
run() { env $3 timeout 600 python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1 $2', round(d['value']), round(d['ms_per_step'],3), 'sel', round(d['kernels']['select']['ms_per_launch']*1e3,1))"; }
for i in 1 2; do run c4 local X=1; done
run c3 local X=1
run c2 local X=1
KVD_TOPK_TRACE=1 timeout 300 python bench.py --config c4 --layers 2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph --fill 1 2>&1 >/dev/null | grep "topk trace" | tail -7
