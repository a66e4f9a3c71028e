#!/bin/bash
# resident-A wide forward (d <= 512): parity + A/B against streamed A (INFCL_FWD_STREAM_A=1), stage counts
mkdir -p gpurun_out
timeout 600 python -m pytest tests/ -m gpu -q --timeout 500 -x > gpurun_out/e39_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e39_pytest.log
for round in 1 2 3; do
  INFCL_FWD_STREAM_A=1 TAG=streamA REPS=9 timeout 120 python scripts/time_step.py
  TAG=resA5 REPS=9 timeout 120 python scripts/time_step.py
  INFCL_STAGES=4 TAG=resA4 REPS=9 timeout 120 python scripts/time_step.py
done > gpurun_out/e39_ab.log 2>&1
for D in 256 384; do
  INFCL_FWD_STREAM_A=1 TAG=streamA_d$D D=$D REPS=9 timeout 120 python scripts/time_step.py
  TAG=resA_d$D D=$D REPS=9 timeout 120 python scripts/time_step.py
done >> gpurun_out/e39_ab.log 2>&1
timeout 300 python scripts/experiments/vring_time.py > gpurun_out/e39_vring.log 2>&1
