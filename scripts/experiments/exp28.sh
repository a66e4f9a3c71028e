#!/bin/bash
REPS=1 INFCL_DEBUG_WAITS=1 python scripts/time_step.py 2>&1 | grep -E "kernel|role" | head -40
REPS=1 D=768 INFCL_DEBUG_WAITS=1 python scripts/time_step.py 2>&1 | grep -E "kernel|role" | head -40
