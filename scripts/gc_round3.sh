#!/bin/bash
# fused backward: L2 hints and a no-drain bound; two-pass wait profile for comparison
mkdir -p gpurun_out
echo "== two-pass waits"; INFCL_FUSED_BWD=0 INFCL_DEBUG_WAITS=1 REPS=2 timeout 120 python scripts/prof_step.py 2>&1 | grep -E "BWD|role" | tail -14
for h in 0 1 3 5 7; do echo "== waits hint $h"; INFCL_GC_HINT=$h INFCL_DEBUG_WAITS=1 REPS=2 timeout 120 python scripts/prof_step.py 2>&1 | grep -E "fused|c-|role 1 wait (full|S-issue|sfree|gready)|role 2" | tail -16; done
echo "== waits no-drain"; INFCL_GC_HINT=8 INFCL_DEBUG_WAITS=1 REPS=2 timeout 120 python scripts/prof_step.py 2>&1 | grep -E "fused|c-" | tail -10
for v in "INFCL_GC_HINT=0" "INFCL_GC_HINT=1" "INFCL_GC_HINT=3" "INFCL_GC_HINT=5" "INFCL_GC_HINT=7" "INFCL_FUSED_BWD=0"; do
  env $v TAG="$v" REPS=9 timeout 120 python scripts/time_step.py 2>&1 | tail -1
done
