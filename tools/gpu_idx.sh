#!/bin/bash
# index / window-scaling iteration: GPU parity + c4h / c3h lines.  usage: tools/gpu_idx.sh <tag>
tag=${1:-ix}; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/${tag}_pytest_gpu.log
for c in c4h c4 c3h; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/${tag}_$c.json 2>gpurun_out/${tag}_$c.err; echo -n "$c: "; python tools/line_summary.py gpurun_out/${tag}_$c.json; tail -2 gpurun_out/${tag}_$c.err
done
