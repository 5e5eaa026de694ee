#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3
for c in c2 c3 c4; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sel_$c.json 2>gpurun_out/sel_$c.err
  python -c "import json; d=json.loads(open('gpurun_out/sel_$c.json').read().strip().splitlines()[-1]); k=d['kernels']; print('$c tok/s %.0f ms %.3f | sel %.1f us %.0f GB/s attn %.1f us res+f %.1f us' % (d['value'], d['ms_per_step'], k['select']['ms_per_launch']*1e3, k['select']['gbs'], k['attn']['ms_per_launch']*1e3, k['resolve_fetch']['ms_per_launch']*1e3))" || tail -3 gpurun_out/sel_$c.err
done
