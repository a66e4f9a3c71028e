#!/bin/bash
mkdir -p gpurun_out
for v in "INFCL_GC_HINT=5" "INFCL_GC_HINT=21" "INFCL_GC_HINT=4" "INFCL_GC_HINT=7" "INFCL_FUSED_BWD=0" "INFCL_GC_HINT=5 INFCL_GC_CONSUMERS=21" "INFCL_GC_HINT=5 INFCL_GC_CONSUMERS=23"; do
  env $v TAG="$v" timeout 120 python scripts/experiments/energy.py 2>&1 | tail -1
done
for h in 5 21; do
INFCL_GC_HINT=$h timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:pair_kernel -c 1 python scripts/prof_step.py 2>&1 | grep -E "dram__|lts__|gpu__time|sm__" | head -8
done
INFCL_DEBUG_WAITS=1 REPS=2 timeout 120 python scripts/prof_step.py 2>&1 | grep -E "fused|c-|role 1" | tail -16
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "bitwise or independent or paired or ragged" > gpurun_out/gc_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gc_pytest.log
