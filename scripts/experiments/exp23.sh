#!/bin/bash
INFCL_LIB=variants/libinfcl_batch.so python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for round in 1 2; do
  TAG=base REPS=9 python scripts/time_step.py
  INFCL_LIB=variants/libinfcl_batch.so TAG=batch REPS=9 python scripts/time_step.py
done
for mode in "" "INFCL_DEBUG_NOEPI=1"; do
  echo "== mode: $mode"
  env $mode REPS=1 INFCL_DEBUG_WAITS=1 python scripts/time_step.py 2>&1 | grep -E "FWD kernel: mean" | head -9
  env $mode REPS=1 INFCL_DEBUG_WAITS=1 INFCL_LIB=variants/libinfcl_batch.so python scripts/time_step.py 2>&1 | grep -E "FWD kernel: mean|role 1" | head -9
done
