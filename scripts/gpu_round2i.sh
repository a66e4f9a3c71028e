#!/bin/bash
# Round-2 final GPU check i (consumer tie-break): full -m gpu suite, smoke, bench (cfg2) + reference arm, ncu launch list of the bench
# command, ncu --set full of the fused backward and the wide forward (one launch each)
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=5 > gpurun_out/gputest_i.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_i.log
tail -9 gpurun_out/gputest_i.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_i.json 2> gpurun_out/bench_i.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_i.json 2>&1; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_i.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_i.log 2>&1; echo "ncu list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:pair_kernel -c 1 -o gpurun_out/prof_r02i_bwd -f \
  python scripts/prof_step.py > gpurun_out/ncu_i2.log 2>&1; echo "ncu bwd rc=$?"
ncu --set full --clock-control none --import-source on -k regex:wide_fwd -c 1 -o gpurun_out/prof_r02i_fwd -f \
  python scripts/prof_step.py > gpurun_out/ncu_i3.log 2>&1; echo "ncu fwd rc=$?"
bash scripts/sweep_b_r02f.sh > gpurun_out/sweep_i.log 2>&1; tail -12 gpurun_out/sweep_i.log
