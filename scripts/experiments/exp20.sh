#!/bin/bash
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for round in 1 2 3; do
  TAG=sbox1 REPS=9 python scripts/time_step.py
  INFCL_SBOX=2 TAG=sbox2 REPS=9 python scripts/time_step.py
done
for round in 1 2; do
  D=768 TAG=sbox1 REPS=5 python scripts/time_step.py
  D=768 INFCL_SBOX=2 TAG=sbox2 REPS=5 python scripts/time_step.py
done
REPS=2 INFCL_DEBUG_WAITS=1 python scripts/time_step.py 2>&1 | grep -v "^{" | head -12
