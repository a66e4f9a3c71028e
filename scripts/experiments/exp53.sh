#!/bin/bash
# deterministic tail (per-pair scratch + pair-ordered combine): determinism, parity suite, A/B step time
mkdir -p gpurun_out
timeout 300 python scripts/experiments/determinism.py > gpurun_out/e54_det.json 2>&1
timeout 1200 python -m pytest tests/ -m gpu -q --timeout 600 -x -rf > gpurun_out/e54_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e54_pytest.log
VARS="prev new" REPS=9 timeout 400 bash scripts/ab.sh > gpurun_out/e54_ab.log 2>&1
for round in 1 2; do for v in prev new; do
  if [ $v = new ]; then L=""; else L=variants/libinfcl_prev.so; fi
  INFCL_LIB=$L B=19244 REPS=9 TAG=${v}_b19244 timeout 120 python scripts/time_step.py
done; done >> gpurun_out/e54_ab.log 2>&1
