#!/bin/bash
# attention pieces-per-segment cap sweep (KVD_ATTN_MAXP) on c2 / c3 / c4
run() { # cfg name env args
  env $3 timeout 600 python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $4 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1 $2', round(d['value']), round(d['ms_per_step'],3), 'attn', round(d['kernels']['attn']['ms_per_launch']*1e3,1))"
}
for m in 32 16 8 4; do
run c2 maxp$m KVD_ATTN_MAXP=$m ""
run c4 maxp$m KVD_ATTN_MAXP=$m ""
run c3 maxp$m KVD_ATTN_MAXP=$m ""
done
