#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -x -q -k "not cfg3 and not onehot_closed_form" 2>&1 | tail -2
for round in 1 2 3; do
  INFCL_LIB=variants/libinfcl_prev.so TAG=prev REPS=9 python scripts/time_step.py
  TAG=new REPS=9 python scripts/time_step.py
  INFCL_BWD_NBUF1=1 TAG=new_nbuf1 REPS=9 python scripts/time_step.py
done
timeout 600 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/bench_e2e3.json 2> gpurun_out/bench_e2e3.err; tail -1 gpurun_out/bench_e2e3.err
