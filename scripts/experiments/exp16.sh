#!/bin/bash
REPS=7 TAG=base python scripts/time_step.py
REPS=3 INFCL_DEBUG_WAITS=1 python scripts/time_step.py 2>&1 | grep -E "FWD kernel|role" | head -9
REPS=7 TAG=base768 D=768 python scripts/time_step.py
