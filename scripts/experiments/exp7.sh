#!/bin/bash
python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 2>&1 | tail -3
for D in 512 768; do TAG=fwd16x256 D=$D python scripts/time_step.py; done
INFCL_DEBUG_WAITS=1 python scripts/time_step.py 2>&1 | grep -E "FWD|role" | head -8
