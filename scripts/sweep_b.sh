#!/bin/bash
# Throughput and peak memory vs global batch at n=1 (BASELINE metric "samples/s and peak GB/GPU vs batch")
mkdir -p gpurun_out
for cfg in "65536 512 20" "131072 512 8" "262144 512 4" "524288 512 3" "1048576 512 3" "65536 768 20" "262144 768 4" "1048576 768 3"; do
  set -- $cfg
  timeout 900 python bench.py --b $1 --d $2 --steps $3 --warmup 3 --no-cpu-baseline 2>>gpurun_out/sweep_b.err | tail -1 >> gpurun_out/sweep_b.jsonl
done
echo done >> gpurun_out/sweep_b.err
