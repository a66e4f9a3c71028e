#!/bin/bash
python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 2>&1 | tail -2
for D in 512 768; do TAG=perwarp D=$D python scripts/time_step.py; done
