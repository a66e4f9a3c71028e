#!/bin/bash
python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -x -q -k "not e2e_host_entry_chunked" 2>&1 | tail -2
VARS="prev new" REPS=9 bash scripts/ab.sh
VARS="prev new" D=768 REPS=5 bash scripts/ab.sh
python scripts/experiments/walk_probe4.py
