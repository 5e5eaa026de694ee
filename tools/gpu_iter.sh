#!/bin/bash
# quick iteration: GPU parity + bench c2/c3/c4 lines.  usage: tools/gpu_iter.sh <tag> [extra bench args]
tag=${1:-it}; shift
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/${tag}_pytest.log | grep -v "^$" | tail -8
for c in c2 c3 c4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline "$@" > gpurun_out/${tag}_bench_$c.json 2> gpurun_out/${tag}_bench_$c.err; echo "$c rc $?"
  python - gpurun_out/${tag}_bench_$c.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    k=d["kernels"]
    print(d["config"]["workload"], "tok/s %.0f ms/step %.3f e2e %.0f hit %.3f launches %s" % (d["value"], d["ms_per_step"], (d["e2e"] or {}).get("value",0), d["hit_rate"], d["gpu_launches"]),
      "| sel %.1fus %.0fGB/s | res+fetch %.1fus | attn %.1fus %.0fGB/s" % (k["select"]["ms_per_launch"]*1e3, k["select"]["gbs"], k["resolve_fetch"]["ms_per_launch"]*1e3, k["attn"]["ms_per_launch"]*1e3, k["attn"]["gbs"]), "clk", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
except Exception as e: print("parse fail", e)
PY
  tail -3 gpurun_out/${tag}_bench_$c.err
done
