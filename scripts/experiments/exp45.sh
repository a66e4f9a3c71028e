#!/bin/bash
# round check after the IPC transport: whole GPU suite (incl. the cfg3-sized IPC ring), smoke, bench, launch list
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -m gpu -q --timeout 600 -rf --durations=6 > gpurun_out/e45_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e45_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e45_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/e45_smoke.log
timeout 600 python bench.py > gpurun_out/e45_bench.json 2> gpurun_out/e45_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e45_launches.csv \
   python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/e45_ncu_bench.log 2>&1
