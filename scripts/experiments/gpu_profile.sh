#!/bin/bash
# ncu evidence for the round: launch list of one bench run and a full-set capture of the two pair kernels.
TAG=${TAG:-r01}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
   python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -c 3 \
   -o gpurun_out/prof_${TAG} -f python scripts/prof_step.py > gpurun_out/ncu_full_${TAG}.log 2>&1
echo done
