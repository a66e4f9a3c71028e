#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -x -q -k "not cfg3 and not onehot_closed_form and not cfg2" 2>&1 | tail -2
VARS="prev new" REPS=9 bash scripts/ab.sh
VARS="prev new" D=768 REPS=5 bash scripts/ab.sh
