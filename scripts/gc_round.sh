#!/bin/bash
# fused backward: correctness vs the two-pass path and the oracle, GPU parity subset, then timing
mkdir -p gpurun_out
TAG=fused timeout 300 python scripts/experiments/gc_check.py > gpurun_out/gc_fused.log 2>&1; echo "fused rc=$?"; tail -12 gpurun_out/gc_fused.log
TAG=twopass INFCL_FUSED_BWD=0 timeout 300 python scripts/experiments/gc_check.py > gpurun_out/gc_twopass.log 2>&1; echo "twopass rc=$?"; tail -3 gpurun_out/gc_twopass.log
CMP=1 timeout 300 python scripts/experiments/gc_check.py 2>&1 | tail -12
for v in "" "INFCL_FUSED_BWD=0" "INFCL_GC_CONSUMERS=18" "INFCL_GC_CONSUMERS=20" "INFCL_GC_CONSUMERS=24" "INFCL_GC_CONSUMERS=26"; do
  env $v TAG="$v" REPS=9 timeout 120 python scripts/time_step.py 2>&1 | tail -1
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ntxent.py -x -q > gpurun_out/gc_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/gc_pytest.log
