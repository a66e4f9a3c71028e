#!/bin/bash
# forward epilogue A/B: two-input max baseline vs FMNMX3 (in-tree) vs FMNMX3 + polynomial exp2 on 1/8, 2/8 of the rows' exps
mkdir -p gpurun_out
python scripts/build_variant.py nofmax3 -DINFCL_FWD_FMAX3=0 > /dev/null 2>&1 &
python scripts/build_variant.py poly1 -DINFCL_FWD_POLY=1 > /dev/null 2>&1 &
python scripts/build_variant.py poly2 -DINFCL_FWD_POLY=2 > /dev/null 2>&1 &
wait; ls variants/
VARS="nofmax3 new poly1 poly2" REPS=9 bash scripts/ab.sh 2>&1 | grep -v Warn
INFCL_LIB=variants/libinfcl_poly2.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "independent or paired or scales" 2>&1 | tail -2
for v in nofmax3 poly2; do INFCL_LIB=variants/libinfcl_$v.so timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__issue_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:wide_fwd -c 1 python scripts/prof_step.py 2>&1 | grep -E "gpu__time|sm__" ; done
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__issue_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:wide_fwd -c 1 python scripts/prof_step.py 2>&1 | grep -E "gpu__time|sm__"
timeout 600 python -m pytest tests/test_gpu_ntxent.py tests/test_gpu_parity.py -x -q -k "scales or ragged or bitwise" 2>&1 | tail -2
