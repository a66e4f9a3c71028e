#!/bin/bash
# Round-2 GPU check g (threaded oracle in the large tests): full -m gpu suite, smoke, bench (cfg2), d = 768 timing with the tuned split
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=10 > gpurun_out/gputest_g.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_g.log
tail -16 gpurun_out/gputest_g.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_g.json 2> gpurun_out/bench_g.err; echo "bench rc=$?"; cat gpurun_out/bench_g.json
