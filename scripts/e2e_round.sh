#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_large.py -x -q -k "e2e" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "e2e" 2>&1 | tail -2
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_f.json')); print(d['value'], d['ms_per_step'], d['e2e'])"
