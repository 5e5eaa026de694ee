#!/bin/bash
# parity + c2/c3/c4 lines (2 rounds)
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
run() { timeout 600 python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', round(d['value']), round(d['ms_per_step'],3), 'sel', round(d['kernels']['select']['ms_per_launch']*1e3,1), 'attn', round(d['kernels']['attn']['ms_per_launch']*1e3,1))"; }
for i in 1 2; do run c3; run c2; run c4; done
