#!/bin/bash
# merge_cols loads four slots in flight: parity subset, determinism, launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -q -m gpu --timeout 600 -x -k "bitwise or waves or cfg2_full or e2e or virtual or ragged or fp32" > gpurun_out/e58_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e58_pytest.log
timeout 300 python scripts/experiments/determinism.py > gpurun_out/e58_det.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e58_launches.csv \
   python scripts/prof_step.py > /dev/null 2>&1
