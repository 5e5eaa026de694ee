#!/bin/bash
# one ncu --set full capture of selected step kernels.  usage: tools/gpu_full.sh <tag> <config> <kernel-regex> <skip> <count> [layers]
tag=$1; cfg=$2; kre=$3; skip=$4; cnt=$5; layers=${6:-2}
mkdir -p gpurun_out
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k "regex:$kre" -s $skip -c $cnt -o gpurun_out/${tag} -f \
  python bench.py --config $cfg --layers $layers --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}.out 2>&1
echo "full $tag rc $?"
