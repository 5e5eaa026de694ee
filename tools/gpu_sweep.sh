#!/bin/bash
# experiment sweep (experiments build: KVD_* overrides honoured).  usage: tools/gpu_sweep.sh <tag>
tag=${1:-sw}; mkdir -p gpurun_out
KVD_BUILD_EXPERIMENTS=1 python -c "from paper_2605_18071_b200 import build as b; b.build(force=True)" || exit 1
run() { name=$1; shift; env "$@" timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-isolated --steps 10 --warmup 3 $BARGS > gpurun_out/${tag}_$name.json 2>gpurun_out/${tag}_$name.err; echo -n "$name: "; python tools/line_summary.py gpurun_out/${tag}_$name.json; }
BARGS="--config c2"
run c2_np20 X=1
run c2_np16 KVD_ATTN_NP=16
run c2_np32 KVD_ATTN_NP=32
run c2_np8 KVD_ATTN_NP=8
BARGS="--config c3"
run c3_np20 X=1
run c3_np32 KVD_ATTN_NP=32
run c3_np16 KVD_ATTN_NP=16
BARGS="--config c4h"
run c4h_np20 X=1
run c4h_np32 KVD_ATTN_NP=32
