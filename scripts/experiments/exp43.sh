#!/bin/bash
# copy-engine batch copies for the IPC transport: overlap probe + IPC multi-process tests
mkdir -p gpurun_out
timeout 300 python scripts/experiments/overlap_probe.py > gpurun_out/e43_overlap.json 2>&1
timeout 400 python -m pytest tests/test_gpu_ipc_ring.py -q --timeout 150 -rf > gpurun_out/e43_ipc.log 2>&1; echo "rc=$?" >> gpurun_out/e43_ipc.log
