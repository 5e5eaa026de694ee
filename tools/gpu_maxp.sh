#!/bin/bash
run() { # cfg name env args
  env $3 timeout 600 python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $4 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1 $2', round(d['value']), round(d['ms_per_step'],3), 'attn', round(d['kernels']['attn']['ms_per_launch']*1e3,1))"
}
KVD_ATTN_MAXP=64 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "qwen or c1_resident or k_all or fused_k_zero" 2>&1 | tail -1
for i in 1 2; do
run c4 maxp32 X=1 ""
run c4 maxp64 KVD_ATTN_MAXP=64 ""
done
run c2 maxp32 X=1 ""
run c2 maxp64 KVD_ATTN_MAXP=64 ""
