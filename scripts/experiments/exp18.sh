#!/bin/bash
REPS=2 INFCL_DEBUG_WAITS=1 python scripts/time_step.py 2>&1 | grep -v "^{" | head -40
REPS=2 D=768 INFCL_DEBUG_WAITS=1 python scripts/time_step.py 2>&1 | grep -v "^{" | head -40
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -c 2 \
   -o gpurun_out/prof_r01c -f python scripts/prof_step.py > gpurun_out/ncu_full_r01c.log 2>&1
tail -3 gpurun_out/ncu_full_r01c.log
