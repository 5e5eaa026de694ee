KVD_BUILD_EXPERIMENTS=1 python -c "from paper_2605_18071_b200 import build as b; b.build(force=True)" || exit 1
python tools/exp_trace.py --config c4h --chain-size 1 --reps 2 2>&1 | tail -30
