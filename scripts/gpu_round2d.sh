#!/bin/bash
# Round-2 GPU check d: full -m gpu suite with the fused backward default, smoke, bench, launch list, ncu of the fused kernel
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=10 > gpurun_out/gputest_d.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_d.log
tail -15 gpurun_out/gputest_d.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_d.json 2> gpurun_out/bench_d.err; echo "bench rc=$?"; cat gpurun_out/bench_d.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:pair_kernel|wide_fwd' -c 2 -o gpurun_out/prof_r02_final python scripts/prof_step.py > gpurun_out/ncu_final.log 2>&1; echo "ncu full rc=$?"
