#!/bin/bash
# c4 / c2 select geometry + attention traces (experiments build).  usage: tools/gpu_c4geo.sh <tag>
tag=${1:-geo}; mkdir -p gpurun_out
KVD_BUILD_EXPERIMENTS=1 python -c "from paper_2605_18071_b200 import build as b; b.build(force=True)" || exit 1
run() { name=$1; shift; env "$@" timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 $BARGS > gpurun_out/${tag}_$name.json 2>gpurun_out/${tag}_$name.err; echo -n "$name: "; python tools/line_summary.py gpurun_out/${tag}_$name.json; }
BARGS="--config c4"
run c4_def X=1
run c4_nt512 KVD_SELECT_NT_LARGE=512
run c4_ctas16 KVD_SELECT_CTAS=16
run c4_ctas16_nt512 KVD_SELECT_CTAS=16 KVD_SELECT_NT_LARGE=512
run c4_span4k KVD_SELECT_MINSPAN_HOST=4096 KVD_SELECT_NT_LARGE=512
python tools/exp_trace.py --config c2 --chain-size 1 --reps 1 2>&1 | tail -14
python tools/exp_trace.py --config c4 --chain-size 1 --reps 1 2>&1 | tail -14
