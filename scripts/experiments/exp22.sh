#!/bin/bash
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for round in 1 2; do
  INFCL_SBOX=2 INFCL_LIB=variants/libinfcl_prev.so TAG=prev REPS=9 python scripts/time_step.py
  TAG=stageasm REPS=9 python scripts/time_step.py
done
for mode in "" "INFCL_DEBUG_NOTMA=1" "INFCL_DEBUG_NOEPI=1" "INFCL_DEBUG_NOTMA=1 INFCL_DEBUG_NOEPI=1"; do
  echo "== mode: $mode"
  env $mode REPS=1 INFCL_DEBUG_WAITS=1 python scripts/time_step.py 2>&1 | grep -E "kernel: mean|role 1|^\{" | head -9
done
