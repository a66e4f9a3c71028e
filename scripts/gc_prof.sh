#!/bin/bash
# fused backward diagnosis: per-role wait cycles (INFCL_DEBUG_WAITS) and one ncu --set full capture at cfg2
mkdir -p gpurun_out
for v in "" "INFCL_GC_CONSUMERS=26" "INFCL_GC_RING=60"; do
  echo "== $v"; env $v INFCL_DEBUG_WAITS=1 REPS=2 timeout 120 python scripts/prof_step.py 2>&1 | grep -E "fused|c-|store|role" | tail -30
done
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:pair_kernel' -c 1 \
    -o gpurun_out/prof_r02_fused python scripts/prof_step.py > gpurun_out/ncu_fused.log 2>&1; echo "ncu rc=$?"
