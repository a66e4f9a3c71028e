#!/bin/bash
# Round-2 GPU check f (re-entry baseline): full -m gpu suite, smoke, bench (cfg2), d = 768 timing with the tuned split
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=10 > gpurun_out/gputest_f.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_f.log
tail -16 gpurun_out/gputest_f.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err; echo "bench rc=$?"; cat gpurun_out/bench_f.json
for v in "" "INFCL_FUSED_BWD=0"; do env $v TAG="$v d768" D=768 REPS=7 timeout 120 python scripts/time_step.py 2>&1 | tail -1; done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_f.json 2>&1; tail -1 gpurun_out/bench_ref_f.json
