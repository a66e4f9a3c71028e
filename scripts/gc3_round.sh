#!/bin/bash
# three-role fused backward: check vs two-pass and oracle, timing vs the two-role kernel, parity subset
mkdir -p gpurun_out
TAG=fused timeout 300 python scripts/experiments/gc_check.py > gpurun_out/gc_fused.log 2>&1; echo "fused rc=$?"; tail -8 gpurun_out/gc_fused.log
TAG=twopass INFCL_FUSED_BWD=0 timeout 300 python scripts/experiments/gc_check.py > gpurun_out/gc_twopass.log 2>&1; echo "twopass rc=$?"
CMP=1 timeout 300 python scripts/experiments/gc_check.py 2>&1 | tail -8
for v in "" "INFCL_BWD3=0" "INFCL_BWD3_P=23" "INFCL_BWD3_P=26" "INFCL_FUSED_BWD=0"; do
  env $v TAG="$v" timeout 120 python scripts/experiments/energy.py 2>&1 | tail -1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ntxent.py -x -q > gpurun_out/gc_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/gc_pytest.log
