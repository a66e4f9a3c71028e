#!/bin/bash
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -c 1 -o gpurun_out/prof_fwd -f python scripts/prof_step.py > gpurun_out/ncu_fwd.log 2>&1
python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "grad_scale" 2>&1 | tail -1
