#!/bin/bash
# quick check: GPU parity (fast tests), c2 per-kernel numbers, attention phase trace
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/q_c2.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/q_c2.json').read().strip().splitlines()[-1]); k=d['kernels']; print('c2 tok/s %.0f ms %.3f | sel %.1f us attn %.1f us res %.1f us' % (d['value'], d['ms_per_step'], k['select']['ms_per_launch']*1e3, k['attn']['ms_per_launch']*1e3, k['resolve_fetch']['ms_per_launch']*1e3))"
KVD_ATTN_TRACE=1 timeout 300 python bench.py --config c2 --layers 2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --chains 1 --no-graph 2>&1 >/dev/null | grep "attn trace" | tail -7
