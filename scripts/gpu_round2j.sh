#!/bin/bash
# Round-2 final GPU check j (final: split ratio 2.2, fused from 16K rows): full -m gpu suite, smoke, bench (cfg2) + reference arm, ncu launch list of the bench
# command, ncu --set full of the fused backward and the wide forward (one launch each)
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=5 > gpurun_out/gputest_j.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_j.log
tail -9 gpurun_out/gputest_j.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_j.json 2> gpurun_out/bench_j.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_j.json 2>&1; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_j.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_j.log 2>&1; echo "ncu list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:pair_kernel -c 1 -o gpurun_out/prof_r02j_bwd -f \
  python scripts/prof_step.py > gpurun_out/ncu_j2.log 2>&1; echo "ncu bwd rc=$?"
ncu --set full --clock-control none --import-source on -k regex:wide_fwd -c 1 -o gpurun_out/prof_r02j_fwd -f \
  python scripts/prof_step.py > gpurun_out/ncu_j3.log 2>&1; echo "ncu fwd rc=$?"
bash scripts/sweep_b_r02j.sh > gpurun_out/sweep_j.log 2>&1; tail -12 gpurun_out/sweep_j.log
