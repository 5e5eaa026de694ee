#!/bin/bash
# SFC chain sweep for c3 / c2
mkdir -p gpurun_out
for m in 4 8 16; do
  timeout 600 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --chains $m > gpurun_out/ch_c3_$m.json 2> gpurun_out/ch_c3_$m.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/ch_c3_$m.json').read().strip().splitlines()[-1]); print('c3 chains', $m, 'tok/s %.0f ms %.3f hit %.3f' % (d['value'], d['ms_per_step'], d['hit_rate']))" || tail -3 gpurun_out/ch_c3_$m.err
done
for m in 1; do
  timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --chains $m > gpurun_out/ch_c2_$m.json 2> gpurun_out/ch_c2_$m.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/ch_c2_$m.json').read().strip().splitlines()[-1]); print('c2 chains', $m, 'tok/s %.0f ms %.3f' % (d['value'], d['ms_per_step']))" || tail -3 gpurun_out/ch_c2_$m.err
done
