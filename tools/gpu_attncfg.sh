#!/bin/bash
for cfg in 1 2 3; do
  KVD_ATTN_CFG=$cfg timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ac_$cfg.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ac_$cfg.json').read().strip().splitlines()[-1]); k=d['kernels']; print('cfg=$cfg c2 tok/s %.0f attn %.1f us' % (d['value'], k['attn']['ms_per_launch']*1e3))"
  KVD_ATTN_CFG=$cfg timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --chains 1 --fill 8 > gpurun_out/ac3_$cfg.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ac3_$cfg.json').read().strip().splitlines()[-1]); k=d['kernels']; print('cfg=$cfg c3 attn %.1f us' % (k['attn']['ms_per_launch']*1e3))"
done
KVD_ATTN_CFG=2 KVD_ATTN_TRACE=1 timeout 300 python bench.py --config c2 --layers 2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --chains 1 --no-graph 2>&1 >/dev/null | grep "attn trace" | tail -7
