#!/bin/bash
INFCL_DEBUG_WAITS=1 python scripts/time_step.py 2>&1 | grep -E "fwd_ms|FWD kernel|BWD kernel|role 1" | head -12
