#!/bin/bash
mkdir -p gpurun_out
for v in "INFCL_BWD3=1" "INFCL_BWD3=0"; do
env $v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum,l1tex__data_pipe_tc_wavefronts_mem_shared.sum,sm__inst_executed.sum --clock-control none -k 'regex:pair_kernel|bwd3' -c 1 python scripts/prof_step.py 2>&1 | grep -E "dram__|lts__|gpu__time|sm__|l1tex" | head -10
done
