#!/bin/bash
# three-role backward: timing vs two-role, and per-role wait counters (INFCL_DEBUG_WAITS)
for r in 1 2; do
  TAG=two-role REPS=7 python scripts/time_step.py
  INFCL_BWD3=1 TAG=three-role REPS=7 python scripts/time_step.py
done
INFCL_BWD3=1 INFCL_DEBUG_WAITS=1 TAG=three-role-dbg REPS=2 python scripts/time_step.py 2>&1 | grep -A30 "bwd3" | tail -32
INFCL_DEBUG_WAITS=1 TAG=two-role-dbg REPS=2 python scripts/time_step.py 2>&1 | grep "dbg" | tail -30
