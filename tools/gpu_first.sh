#!/bin/bash
# first GPU pass of a round: box facts, GPU parity, bench lines
mkdir -p gpurun_out
bash tools/box_probe.sh
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config c2 --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc $?"
timeout 900 python bench.py --config c3 --steps 10 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc $?"
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench_c2.json gpurun_out/bench_c3.json; tail -5 gpurun_out/bench_c2.err gpurun_out/bench_c3.err
