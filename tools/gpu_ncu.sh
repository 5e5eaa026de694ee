#!/bin/bash
# ncu evidence for the bench: launch lists (same command as the bench, steady-state
# launches only) and one --set full capture of each step kernel (2-layer copy of c3/c2:
# per-layer kernels are identical in shape; keeps ncu's replay memory small).
# usage: tools/gpu_ncu.sh <tag>
tag=${1:-r01}
mkdir -p gpurun_out
K='regex:score_kernel|topk_kernel|resolve_kernel|gather_kernel|attn_kernel'
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" -s 5120 -c 320 --csv \
  --log-file gpurun_out/${tag}_launches_c3.csv python bench.py --config c3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_ncu_c3.out 2>&1
echo "launches c3 rc $?"
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" -s 128 -c 256 --csv \
  --log-file gpurun_out/${tag}_launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_ncu_c2.out 2>&1
echo "launches c2 rc $?"
timeout 900 $NCU --set full --clock-control none --import-source on -k "$K" -s 320 -c 5 -o gpurun_out/${tag}_full_c3 -f \
  python bench.py --config c3 --layers 2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_full_c3.out 2>&1
echo "full c3 rc $?"
timeout 600 $NCU --set full --clock-control none --import-source on -k "$K" -s 8 -c 4 -o gpurun_out/${tag}_full_c2 -f \
  python bench.py --config c2 --layers 2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_full_c2.out 2>&1
echo "full c2 rc $?"
ls -la gpurun_out
