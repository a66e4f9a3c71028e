#!/bin/bash
mkdir -p gpurun_out
for v in "INFCL_GC_HINT=0" "INFCL_GC_HINT=1" "INFCL_GC_HINT=3" "INFCL_GC_HINT=5" "INFCL_FUSED_BWD=0" "INFCL_GC_RING=24" "INFCL_GC_RING=28"; do
  env $v TAG="$v" timeout 120 python scripts/experiments/energy.py 2>&1 | tail -1
done
for h in 0 5; do
INFCL_GC_HINT=$h timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:pair_kernel -c 1 python scripts/prof_step.py 2>&1 | grep -E "pair_kernel|dram__|lts__|gpu__time|sm__" | head -8
done
