#!/bin/bash
python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -x -q -k "e2e or parity_paired or independent" 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; tail -2 gpurun_out/bench_e2e.err
