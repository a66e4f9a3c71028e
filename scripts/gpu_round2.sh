#!/bin/bash
# Round-2 GPU check: full -m gpu suite, bench N=1, the N=2 path check on one GPU (self-spawned ranks).
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
tail -30 gpurun_out/gputest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json
INFCL_BENCH_SAME_GPU=1 timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n2_samegpu.json 2> gpurun_out/bench_n2.err; echo "n2 rc=$?"
cat gpurun_out/bench_n2_samegpu.json; tail -5 gpurun_out/bench_n2.err
