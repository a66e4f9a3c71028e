#!/bin/bash
# IPC ring transport after the comm-stream arrival fix: multi-process ring on one GPU, bench N=2/3 path on
# one GPU (ranks share cuda:0; not a throughput number), then the whole GPU suite
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_ipc_ring.py -q --timeout 150 -rf > gpurun_out/e42_ipc.log 2>&1; echo "rc=$?" >> gpurun_out/e42_ipc.log
for N in 2 3; do
INFCL_BENCH_SAME_GPU=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
  --master-port 2955$N bench.py --gpus $N --steps 3 --warmup 3 --b $((12288*N)) > gpurun_out/e42_bench$N.json 2> gpurun_out/e42_bench$N.err; echo "rc=$?" >> gpurun_out/e42_bench$N.err
done
timeout 900 python -m pytest tests/ -m gpu -q --timeout 400 -rf > gpurun_out/e42_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e42_pytest.log
