#!/bin/bash
# experiment sweep (experiments build: KVD_* overrides honoured).
# usage: tools/gpu_sweep.sh <tag> "<name>|<bench args>|<env>" ...
tag=${1:-sw}; shift; mkdir -p gpurun_out
KVD_BUILD_EXPERIMENTS=1 python -c "from paper_2605_18071_b200 import build as b; b.build(force=True)" || exit 1
for spec in "$@"; do
  IFS='|' read -r name bargs envs <<< "$spec"
  env X=1 $envs timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-isolated --steps 10 --warmup 3 $bargs \
    > gpurun_out/${tag}_$name.json 2>gpurun_out/${tag}_$name.err
  echo -n "$name: "; python tools/line_summary.py gpurun_out/${tag}_$name.json
done
