#!/bin/bash
for round in 1 2; do
  TAG=st4 REPS=7 python scripts/time_step.py
  INFCL_STAGES=3 TAG=st3 REPS=7 python scripts/time_step.py
  INFCL_STAGES=2 TAG=st2 REPS=7 python scripts/time_step.py
done
