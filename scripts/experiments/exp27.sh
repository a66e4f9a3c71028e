#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -4
for round in 1 2; do
  TAG=wide REPS=9 python scripts/time_step.py
  INFCL_FWD_NARROW=1 TAG=narrow REPS=9 python scripts/time_step.py
done
D=768 TAG=wide REPS=5 python scripts/time_step.py
D=768 INFCL_FWD_NARROW=1 TAG=narrow REPS=5 python scripts/time_step.py
REPS=1 INFCL_DEBUG_WAITS=1 python scripts/time_step.py 2>&1 | grep -E "FWD|role" | head -12
