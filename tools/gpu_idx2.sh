#!/bin/bash
tag=${1:-ix}; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -k "index or window or c4h" > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/${tag}_pytest_gpu.log
for c in c4h; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/${tag}_$c.json 2>gpurun_out/${tag}_$c.err; echo -n "$c: "; python tools/line_summary.py gpurun_out/${tag}_$c.json; tail -2 gpurun_out/${tag}_$c.err
done
bash tools/gpu_trace_idx.sh 2>&1 | grep -A9 cand_kernel | head -10
