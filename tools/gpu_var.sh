#!/bin/bash
# variants: c3 fused gather in/out; c2 chains.
run() { # cfg name env args
  env $3 timeout 600 python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $4 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1 $2', round(d['value']), round(d['ms_per_step'],3))"
}
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fused" 2>&1 | tail -1
KVD_FUSED_GATHER=0 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fused" 2>&1 | tail -1
for i in 1 2; do
run c3 inner X=1 ""
run c3 outer KVD_FUSED_GATHER=0 ""
done
run c2 ch1 X=1 ""
run c2 ch2 X=1 "--chains 2"
run c2 ch4 X=1 "--chains 4"
run c2 ch8 X=1 "--chains 8"
run c4 ch4 X=1 ""
run c4 ch4o KVD_FUSED_GATHER=0 ""
run c4 ch1 X=1 "--chains 1"
run c4 ch2 X=1 "--chains 2"
