#!/bin/bash
# Round-2 GPU check c: the whole -m gpu suite, smoke, bench N=1, ncu --set full at d = 768 (cfg3/n=8 per-rank and b=65536).
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=20 > gpurun_out/gputest_c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_c.log
tail -30 gpurun_out/gputest_c.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_c.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_c.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err; echo "bench rc=$?"
cat gpurun_out/bench_c.json
for cfg in "32768 768" "65536 768"; do
  set -- $cfg
  B=$1 D=$2 timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:pair_kernel|wide_fwd' -c 3 \
    -o gpurun_out/prof_r02_b$1_d$2 python scripts/prof_step.py > gpurun_out/ncu_b$1_d$2.log 2>&1
  echo "ncu $1 $2 rc=$?"
done
