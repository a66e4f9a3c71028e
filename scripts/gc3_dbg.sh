#!/bin/bash
for v in "" "INFCL_BWD3_P=26"; do
echo "== $v"; env $v INFCL_DEBUG_WAITS=1 REPS=2 timeout 120 python scripts/prof_step.py 2>&1 | grep -E "bwd3|prod|dI-|dT-" | tail -30
done
for v in "" "INFCL_BWD3_P=26" "INFCL_BWD3_P=25" "INFCL_BWD3=0"; do
  env $v TAG="$v" timeout 120 python scripts/experiments/energy.py 2>&1 | tail -1
done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "independent or paired or ragged or bitwise or splits" 2>&1 | tail -2
