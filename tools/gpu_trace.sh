#!/bin/bash
# experiments build + phase traces + A/B bench lines.  usage: tools/gpu_trace.sh <tag>
tag=${1:-tr}; mkdir -p gpurun_out
KVD_BUILD_EXPERIMENTS=1 python -c "from paper_2605_18071_b200 import build as b; b.build(force=True)" || exit 1
python tools/exp_trace.py --config c2 --chain-size 1 --reps 2 2>&1 | tail -14
KVD_NO_PREFETCH=1 python tools/exp_trace.py --config c2 --chain-size 1 --reps 1 2>&1 | tail -7
python tools/exp_trace.py --config c3 --chain-size 1 --reps 1 2>&1 | tail -14
run() { name=$1; shift; env "$@" timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 $BARGS > gpurun_out/${tag}_$name.json 2>gpurun_out/${tag}_$name.err; echo -n "$name: "; python tools/line_summary.py gpurun_out/${tag}_$name.json; }
for c in c2 c3 c4; do BARGS="--config $c"; run ${c} X=1; run ${c}_nopf KVD_NO_PREFETCH=1; done
