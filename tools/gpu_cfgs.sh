#!/bin/bash
mkdir -p gpurun_out
for c in c4 c5 c1; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err; echo "$c rc $?"
  python -c "import json; d=json.loads(open('gpurun_out/cfg_$c.json').read().strip().splitlines()[-1]); k=d['kernels']; print('$c tok/s %.0f ms %.3f e2e %.0f hit %.3f setup %.0fs | sel %.1f us attn %.1f us res+f %.1f us | roof %s %.2f' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['hit_rate'], d['setup_s'], k['select']['ms_per_launch']*1e3, k['attn']['ms_per_launch']*1e3, k['resolve_fetch']['ms_per_launch']*1e3, d['roofline']['bound'], d['roofline']['frac']))" || tail -4 gpurun_out/cfg_$c.err
done
timeout 600 python bench.py --config c4 --shard heads --steps 5 --warmup 3 --no-cpu-baseline --fill 8 > gpurun_out/cfg_c4h.json 2> gpurun_out/cfg_c4h.err; echo "c4 heads rc $?"; tail -c 300 gpurun_out/cfg_c4h.json; tail -3 gpurun_out/cfg_c4h.err
K="regex:score_kernel|topk_kernel|resolve_kernel|gather_kernel|attn_kernel"
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" \
  -s $((2*2048 + 3*2048)) -c 2048 --csv --log-file gpurun_out/r01_launches_default.csv python bench.py --steps 2 --warmup 3 --fill 2 --no-e2e --no-cpu-baseline > gpurun_out/r01_ncu_default.out 2>&1
echo "launch list rc $?"
python tools/ncu_summary.py gpurun_out/r01_launches_default.csv
