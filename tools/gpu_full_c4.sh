#!/bin/bash
K="regex:score_kernel|topk_kernel|resolve_kernel|gather_kernel|attn_kernel|merge_kernel"
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k "$K" -s 4 -c 8 -o gpurun_out/r01e_full_c4 -f \
  python bench.py --config c4 --layers 2 --chains 1 --no-graph --fill 1 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r01e_full_c4.out 2>&1
echo "full c4 rc $?"
