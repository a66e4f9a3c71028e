#!/bin/bash
# diag-init + merge_cols(G=32) check: gpu parity, TMA probe 3, A/B step time, virtual ring timing
mkdir -p gpurun_out
timeout 600 python -m pytest tests/ -m gpu -q --timeout 500 -x > gpurun_out/e38_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e38_pytest.log
timeout 120 python scripts/experiments/tma_rate3.py > gpurun_out/e38_tma3.log 2>&1
VARS="prev new" REPS=9 timeout 300 bash scripts/ab.sh > gpurun_out/e38_ab.log 2>&1
timeout 300 python scripts/experiments/vring_time.py > gpurun_out/e38_vring.log 2>&1
INFCL_LIB=variants/libinfcl_prev.so timeout 300 python scripts/experiments/vring_time.py > gpurun_out/e38_vring_prev.log 2>&1
