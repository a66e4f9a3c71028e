#!/bin/bash
# fused backward v2 (epilogue G writes, transposed consumer, unified ring, v4 drains): check, waits, timing, parity
mkdir -p gpurun_out
TAG=fused timeout 300 python scripts/experiments/gc_check.py > gpurun_out/gc_fused.log 2>&1; echo "fused rc=$?"; tail -8 gpurun_out/gc_fused.log
TAG=twopass INFCL_FUSED_BWD=0 timeout 300 python scripts/experiments/gc_check.py > gpurun_out/gc_twopass.log 2>&1; echo "twopass rc=$?"
CMP=1 timeout 300 python scripts/experiments/gc_check.py 2>&1 | tail -8
INFCL_DEBUG_WAITS=1 REPS=2 timeout 120 python scripts/prof_step.py 2>&1 | grep -E "fused|c-|role" | tail -30
for v in "" "INFCL_GC_CONSUMERS=18" "INFCL_GC_CONSUMERS=20" "INFCL_GC_CONSUMERS=24" "INFCL_FUSED_BWD=0"; do
  env $v TAG="$v" REPS=9 timeout 120 python scripts/time_step.py 2>&1 | tail -1
done
for v in "" "INFCL_FUSED_BWD=0"; do
  env $v TAG="$v d768" D=768 REPS=5 timeout 120 python scripts/time_step.py 2>&1 | tail -1
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ntxent.py -x -q > gpurun_out/gc_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/gc_pytest.log
