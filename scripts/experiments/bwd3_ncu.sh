#!/bin/bash
# ncu source-level capture of the three-role backward (one launch)
mkdir -p gpurun_out
INFCL_BWD3=1 timeout 600 ncu --section SourceCounters --section WarpStateStats --section SpeedOfLight --clock-control none \
  --import-source on -k regex:bwd3 -c 1 -o gpurun_out/bwd3_src -f python scripts/prof_step.py > gpurun_out/bwd3_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/bwd3_ncu.log
ncu -i gpurun_out/bwd3_src.ncu-rep --page source --csv --print-source sass > gpurun_out/bwd3_src_sass.csv 2>/dev/null
ncu -i gpurun_out/bwd3_src.ncu-rep --page source --csv --print-source cuda > gpurun_out/bwd3_src_cuda.csv 2>/dev/null
ls -la gpurun_out/bwd3_src*
