#!/bin/bash
# fused backward ring (world > 1): virtual ring, multi-process IPC ring on one GPU, large virtual-ring protocols,
# bench path check at N = 2 (same GPU)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ipc_ring.py -x -q -k "virtual or ipc" > gpurun_out/ring_pytest.log 2>&1; echo "pytest ring rc=$?"; tail -4 gpurun_out/ring_pytest.log
timeout 1500 python -m pytest tests/test_gpu_large.py -x -q > gpurun_out/ring_large.log 2>&1; echo "pytest large rc=$?"; tail -4 gpurun_out/ring_large.log
INFCL_BENCH_SAME_GPU=1 timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n2_fused.json 2> gpurun_out/bench_n2_fused.err; echo "n2 rc=$?"; cat gpurun_out/bench_n2_fused.json | head -c 1500; echo
INFCL_FUSED_RING=0 INFCL_BENCH_SAME_GPU=1 timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n2_twopass.json 2> gpurun_out/bench_n2_tp.err; echo "n2 tp rc=$?"; python -c "import json; d=json.load(open('gpurun_out/bench_n2_twopass.json')); print(d['ms_per_step'], d['bwd_ms'])"
