#!/bin/bash
# three-role backward A/B vs the two-role default; optional parity
if [ -n "$PARITY" ]; then timeout 600 python -m pytest tests/test_gpu_parity.py -q -k three_role 2>&1 | tail -2; fi
for r in 1 2; do
  TAG=two-role REPS=7 python scripts/time_step.py
  INFCL_BWD3=1 TAG=three-role REPS=7 python scripts/time_step.py
done
INFCL_BWD3=1 INFCL_DEBUG_WAITS=1 TAG=three-role-dbg REPS=2 python scripts/time_step.py 2>&1 | grep -A30 "bwd3:" | grep -v "^{" | head -30
