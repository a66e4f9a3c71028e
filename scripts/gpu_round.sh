#!/bin/bash
# Full round check on one GPU: tests, smoke, launch list + ncu full capture, bench (TAG names the profile files)
TAG=${TAG:-r01d}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -m gpu -q --timeout 900 -rf --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?" >> gpurun_out/bench_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
   python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pair_kernel|wide_fwd" -c 2 \
   -o gpurun_out/prof_${TAG} -f python scripts/prof_step.py > gpurun_out/ncu_full_${TAG}.log 2>&1
echo done
