#!/bin/bash
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
VARS="prev hint new" bash scripts/ab.sh
VARS="prev new" D=768 REPS=5 bash scripts/ab.sh
