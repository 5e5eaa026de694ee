#!/bin/bash
# A/B on one box: abtest/ (older build) vs the working tree, c3 and c2, alternating.
for i in 1 2; do
for c in c3 c2 c4; do
  (cd abtest && timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('A(old) $c', round(d['value']), round(d['ms_per_step'],3))")
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('B(new) $c', round(d['value']), round(d['ms_per_step'],3))"
done
done
