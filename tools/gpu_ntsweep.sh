#!/bin/bash
# top-k CTA size sweep (KVD_TOPK_THREADS) on c2 / c3 / c4.  usage: tools/gpu_ntsweep.sh <tag>
tag=${1:-nt}; mkdir -p gpurun_out
for nt in 256 512 1024; do
  KVD_TOPK_THREADS=$nt timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "topk or c1_resident or ragged" 2>&1 | tail -1
  for c in c3 c2 c4; do
    KVD_TOPK_THREADS=$nt timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_${c}_$nt.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/${tag}_${c}_$nt.json').read().strip().splitlines()[-1]);print('$c nt=$nt', round(d['value']), round(d['ms_per_step'],3), 'sel', round(d['kernels']['select']['ms_per_launch']*1e3,1), 'attn', round(d['kernels']['attn']['ms_per_launch']*1e3,1), 'res', round(d['kernels']['resolve_fetch']['ms_per_launch']*1e3,1))" 2>&1 | tail -1
  done
done
