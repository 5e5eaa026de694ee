#!/bin/bash
run() { env $3 timeout 600 python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1 $2', round(d['value']), round(d['ms_per_step'],3), 'sel', round(d['kernels']['select']['ms_per_launch']*1e3,1))"; }
KVD_TOPK_KPT=8 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "topk or fused" 2>&1 | tail -1
for i in 1 2; do run c4 kpt16 X=1; run c4 kpt8 KVD_TOPK_KPT=8; done
KVD_TOPK_KPT=8 KVD_TOPK_TRACE=1 timeout 300 python bench.py --config c4 --layers 2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --chains 4 --no-graph --fill 1 2>&1 >/dev/null | grep "topk trace" | tail -7
