#!/bin/bash
python scripts/experiments/mma_rate.py 2>&1 | head -3
python scripts/experiments/mma_rate2.py
for D in 512 768; do
 TAG=stage32k D=$D python scripts/time_step.py
 TAG=stage32k_s2 D=$D INFCL_STAGES=2 python scripts/time_step.py
done
python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 2>&1 | tail -2
