#!/bin/bash
python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "e2e or autograd or independent" 2>&1 | tail -2
timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/bench_e2e.json 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum --clock-control none -k regex:pair_kernel -c 3 python scripts/prof_step.py > gpurun_out/ncu_mem.log 2>&1
