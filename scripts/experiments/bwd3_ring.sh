#!/bin/bash
# three-role backward: is the G ring depth (steps in flight) the limiter?  ring = P_c + 12 (38) by default
for r in 1 2; do
  INFCL_BWD3=1 TAG=three-role REPS=5 python scripts/time_step.py
  for R in 64 96; do INFCL_BWD3=1 INFCL_GC_RING=$R TAG="three-role ring $R" REPS=5 python scripts/time_step.py; done
  for P in 22 20; do INFCL_BWD3=1 INFCL_BWD3_P=$P TAG="three-role P=$P" REPS=5 python scripts/time_step.py; done
done
INFCL_BWD3=1 INFCL_GC_RING=96 INFCL_DEBUG_WAITS=1 TAG=dbg REPS=2 python scripts/time_step.py 2>&1 | grep -A30 "bwd3:" | grep -v "^{" | head -30
