#!/bin/bash
# backward with two MMA-issuing warps (S GEMMs / dA GEMMs) vs the previous single issuer (variant prev2):
# parity subset, then interleaved timing at cfg2 and d = 768, fused and two-pass backward
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "not grad_scale_cfg2" 2>&1 | tail -2
for r in 1 2 3; do
  INFCL_LIB=variants/libinfcl_prev2.so TAG=prev REPS=7 python scripts/time_step.py
  TAG=two-issuer REPS=7 python scripts/time_step.py
done
for r in 1 2; do
  INFCL_LIB=variants/libinfcl_prev2.so INFCL_FUSED_BWD=0 TAG="prev two-pass" REPS=7 python scripts/time_step.py
  INFCL_FUSED_BWD=0 TAG="two-issuer two-pass" REPS=7 python scripts/time_step.py
  INFCL_LIB=variants/libinfcl_prev2.so D=768 TAG="prev d768" REPS=5 python scripts/time_step.py
  D=768 TAG="two-issuer d768" REPS=5 python scripts/time_step.py
done
INFCL_DEBUG_WAITS=1 TAG=dbg REPS=2 python scripts/time_step.py 2>&1 | grep "dbg" | tail -30
