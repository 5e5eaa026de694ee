#!/bin/bash
# c3 variants sweep (fused path).  usage: tools/gpu_c3sweep.sh <tag>
tag=${1:-sw}; mkdir -p gpurun_out
run() { # name, env, args
  env $2 timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $3 > gpurun_out/${tag}_$1.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/${tag}_$1.json').read().strip().splitlines()[-1]);print('$1', round(d['value']), round(d['ms_per_step'],3))" 2>&1 | tail -1
}
run base "X=1" ""
run v4 "KVD_SEL_V=4" ""
run ch8 "X=1" "--chains 8"
run nt512 "KVD_TOPK_THREADS=512" ""
run nt256 "KVD_TOPK_THREADS=256" ""
run attn1 "KVD_ATTN_CFG=1" ""
run base2 "X=1" ""
