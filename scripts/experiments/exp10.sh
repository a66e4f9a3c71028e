#!/bin/bash
for v in "" "INFCL_DEBUG_NOEPI=1" "INFCL_DEBUG_NOTMA=1" "INFCL_DEBUG_NOEPI=1 INFCL_DEBUG_NOTMA=1"; do
  echo "== $v"; env $v INFCL_DEBUG_WAITS=1 python scripts/time_step.py 2>&1 | grep -E "fwd_ms|FWD kernel|BWD kernel|role 1 wait (full|sfree|gready)" | head -7
done
