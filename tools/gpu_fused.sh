#!/bin/bash
# fused vs unfused, parity + c2/c3/c4.  usage: tools/gpu_fused.sh <tag>
tag=${1:-fu}; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/${tag}_pytest.log | grep -v "^$" | tail -6
for c in c2 c3 c4; do
 for v in "" "--unfused"; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $v > gpurun_out/${tag}_${c}$v.json 2>gpurun_out/${tag}_${c}$v.err
  python -c "import json;d=json.loads(open('gpurun_out/${tag}_${c}$v.json').read().strip().splitlines()[-1]);print('$c $v', round(d['value']), round(d['ms_per_step'],3), 'launches', d['gpu_launches'])" 2>&1 | tail -1
 done
done
