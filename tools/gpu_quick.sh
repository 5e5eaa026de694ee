#!/bin/bash
# quick GPU iteration: parity suite + bench lines.  usage: tools/gpu_quick.sh <tag> [configs...]
tag=${1:-q}; shift; cfgs=${@:-c3 c2 c4}; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/${tag}_pytest_gpu.log
for cfg in $cfgs; do
  timeout 900 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/${tag}_bench_$cfg.json 2> gpurun_out/${tag}_bench_$cfg.err; echo "$cfg rc $?"
  python tools/line_summary.py gpurun_out/${tag}_bench_$cfg.json
done
