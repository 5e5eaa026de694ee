#!/bin/bash
# c3 / c2 select geometry sweep (experiments build).  usage: tools/gpu_c3geo.sh <tag>
tag=${1:-geo}; mkdir -p gpurun_out
KVD_BUILD_EXPERIMENTS=1 python -c "from paper_2605_18071_b200 import build as b; b.build(force=True)" || exit 1
run() { name=$1; shift; env "$@" timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 $BARGS > gpurun_out/${tag}_$name.json 2>gpurun_out/${tag}_$name.err; echo -n "$name: "; python tools/line_summary.py gpurun_out/${tag}_$name.json; }
BARGS="--config c3"
for t in 8 16 32 64; do run c3_ctas$t KVD_SELECT_CTAS=$t; done
run c3_ctas8_nt1024 KVD_SELECT_CTAS=8 KVD_SELECT_NT_SMALL=1024
BARGS="--config c2"
for t in 8 16 32; do run c2_ctas$t KVD_SELECT_CTAS=$t; done
run c2_nt1024 KVD_SELECT_NT_SMALL=1024
BARGS="--config c4"
for t in 32 128; do run c4_ctas$t KVD_SELECT_CTAS=$t; done
