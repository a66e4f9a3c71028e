#!/bin/bash
# d = 768 (ViT-L/14, the north-star shape): forward ring depth A/B (INFCL_STAGES caps both kernels; the
# backward has 3 stages at d = 768 anyway)
mkdir -p gpurun_out
for round in 1 2; do
  for ns in 6 4 5; do
    INFCL_STAGES=$ns TAG=d768_ns$ns D=768 B=131072 REPS=7 timeout 200 python scripts/time_step.py
  done
done > gpurun_out/e56.log 2>&1
