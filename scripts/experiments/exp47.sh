#!/bin/bash
# fused per-step merge (rows + columns in one launch) and fused forward finish: GPU suite, small-b A/B, vring
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -m gpu -q --timeout 600 -x -rf > gpurun_out/e47_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e47_pytest.log
for round in 1 2; do for v in prev new; do
  if [ $v = new ]; then L=""; else L=variants/libinfcl_prev.so; fi
  for b in 8192 16384; do INFCL_LIB=$L B=$b REPS=15 TAG=${v}_b$b timeout 120 python scripts/time_step.py; done
done; done > gpurun_out/e47_smallb.log 2>&1
timeout 300 python scripts/experiments/vring_time.py > gpurun_out/e47_vring.log 2>&1
INFCL_LIB=variants/libinfcl_prev.so timeout 300 python scripts/experiments/vring_time.py > gpurun_out/e47_vring_prev.log 2>&1
