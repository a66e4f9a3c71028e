#!/bin/bash
# IPC (copy-engine) ring transport: multi-process ring on one GPU, then the whole GPU suite
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_ipc_ring.py -x -q --timeout 150 -rf > gpurun_out/e41_ipc.log 2>&1; echo "rc=$?" >> gpurun_out/e41_ipc.log
timeout 900 python -m pytest tests/ -m gpu -q --timeout 400 -x -rf > gpurun_out/e41_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e41_pytest.log
