#!/bin/bash
# iteration: GPU parity, bench lines, then an experiments build with phase traces.  usage: tools/gpu_iter.sh <tag> [cfgs]
tag=${1:-it}; shift; cfgs=${@:-c2 c3 c4}; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/${tag}_pytest_gpu.log
for c in $cfgs; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/${tag}_$c.json 2>gpurun_out/${tag}_$c.err; echo -n "$c: "; python tools/line_summary.py gpurun_out/${tag}_$c.json
done
KVD_BUILD_EXPERIMENTS=1 python -c "from paper_2605_18071_b200 import build as b; b.build(force=True)" || exit 1
python tools/exp_trace.py --config c2 --chain-size 1 --reps 2 2>&1 | tail -13
python tools/exp_trace.py --config c3 --chain-size 1 --reps 1 2>&1 | tail -13
python tools/exp_trace.py --config c4 --chain-size 1 --reps 1 2>&1 | tail -13
