#!/bin/bash
for x in 0 1 2 3; do
  KVD_ATTN_X=$x timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --chains 1 > gpurun_out/ax_$x.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ax_$x.json').read().strip().splitlines()[-1]); k=d['kernels']; print('x=$x attn %.1f us sel %.1f us' % (k['attn']['ms_per_launch']*1e3, k['select']['ms_per_launch']*1e3))"
done
for st in 3 6; do
  KVD_ATTN_STAGES=$st timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --chains 1 > gpurun_out/as_$st.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/as_$st.json').read().strip().splitlines()[-1]); k=d['kernels']; print('stages=$st attn %.1f us' % (k['attn']['ms_per_launch']*1e3))"
done
