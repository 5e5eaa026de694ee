#!/bin/bash
# ncu --set full of chain-sized select / attention launches (c2, eager, 2 layers).  usage: tools/gpu_ncu_sel.sh <tag>
tag=${1:-ns}; mkdir -p gpurun_out
K="regex:select_kernel|attn_kernel|merge_kernel"
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k "$K" -s 48 -c 6 -o gpurun_out/${tag}_c2 -f \
  python bench.py --config c2 --layers 2 --no-graph --fill 3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_c2.out 2>&1
echo "ncu c2 rc $?"
python tools/ncu_details.py gpurun_out/${tag}_c2.ncu-rep | head -60
