#!/bin/bash
# experiment sweep (experiments build: KVD_* overrides honoured) + ncu captures.  usage: tools/gpu_sweep.sh <tag>
tag=${1:-sw}; mkdir -p gpurun_out
KVD_BUILD_EXPERIMENTS=1 python -c "from paper_2605_18071_b200 import build as b; b.build(force=True)" || exit 1
run() { name=$1; shift; env "$@" timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 $BARGS > gpurun_out/${tag}_$name.json 2>gpurun_out/${tag}_$name.err; echo -n "$name: "; python tools/line_summary.py gpurun_out/${tag}_$name.json; }
BARGS="--config c2"
run c2_def X=1
run c2_pt4 KVD_ATTN_PIECE_TILES=4
run c2_pt16 KVD_ATTN_PIECE_TILES=16
BARGS="--config c2 --chains 1"; run c2_chains1 X=1
BARGS="--config c2 --chains 4"; run c2_chains4 X=1
BARGS="--config c2 --chains 16 --alias 0"; run c2_chains16 X=1
BARGS="--config c3"; run c3_def X=1
BARGS="--config c3"; run c3_ctas256 KVD_SELECT_CTAS=256
BARGS="--config c3"; run c3_ctas16 KVD_SELECT_CTAS=16
BARGS="--config c4"; run c4_def X=1
BARGS="--config c4"; run c4_ctas16 KVD_SELECT_CTAS=16
K="regex:select_kernel|attn_kernel"
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k "$K" -s 8 -c 4 -o gpurun_out/${tag}_full_c2 -f \
  python bench.py --config c2 --layers 2 --chains 8 --no-graph --fill 1 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_full_c2.out 2>&1
echo "ncu c2 rc $?"
python tools/ncu_details.py gpurun_out/${tag}_full_c2.ncu-rep select_kernel attn_kernel > gpurun_out/${tag}_full_c2.txt 2>&1; head -80 gpurun_out/${tag}_full_c2.txt
