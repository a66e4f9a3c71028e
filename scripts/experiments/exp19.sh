#!/bin/bash
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
VARS="prev new" bash scripts/ab.sh
REPS=2 INFCL_DEBUG_WAITS=1 python scripts/time_step.py 2>&1 | grep -v "^{" | head -12
