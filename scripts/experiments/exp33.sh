#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for round in 1 2 3; do
  TAG=pair REPS=9 python scripts/time_step.py
  INFCL_NO_PAIR_COMMIT=1 TAG=nopair REPS=9 python scripts/time_step.py
done
for round in 1 2; do
  D=768 TAG=pair REPS=5 python scripts/time_step.py
  D=768 INFCL_NO_PAIR_COMMIT=1 TAG=nopair REPS=5 python scripts/time_step.py
done
