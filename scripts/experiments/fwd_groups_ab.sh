#!/bin/bash
# Wide-forward epilogue groups A/B: committed build (prev) vs three groups (new) vs two groups in the new layout
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "forward or fwd or random or onehot or scale" 2>&1 | tail -3
for round in 1 2 3; do
  INFCL_LIB=variants/libinfcl_prev.so TAG=prev REPS=9 python scripts/time_step.py
  TAG=ng3 REPS=9 python scripts/time_step.py
  INFCL_FWD_GROUPS=2 TAG=ng2 REPS=9 python scripts/time_step.py
done
for round in 1 2; do
  INFCL_LIB=variants/libinfcl_prev.so TAG="prev d768" D=768 REPS=7 python scripts/time_step.py
  TAG="ng3 d768" D=768 REPS=7 python scripts/time_step.py
done
