#!/bin/bash
# Round-2 GPU check b: the new and changed tests, ncu at d = 768, the bench.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_ntxent.py tests/test_gpu_parity.py "tests/test_gpu_ipc_ring.py::test_ipc_ring_ntxent" \
  "tests/test_gpu_large.py::test_cfg5_random_sampled_protocol" -q --durations=10 > gpurun_out/gputest_b.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest_b.log
tail -25 gpurun_out/gputest_b.log
for cfg in "32768 768" "65536 768"; do
  set -- $cfg
  B=$1 D=$2 timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:pair_kernel|wide_fwd' -c 3 \
    -o gpurun_out/prof_r02_b$1_d$2 python scripts/prof_step.py > gpurun_out/ncu_b$1_d$2.log 2>&1
  echo "ncu $1 $2 rc=$?"
done
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err; echo "bench rc=$?"
cat gpurun_out/bench_b.json
