#!/bin/bash
# plan ratio 2.2 (this build) vs the previous plan (variant prev3: 2.5 at d=512, 2.0 at d=768), interleaved
for r in 1 2; do
  for cfg in "65536 512 7" "262144 512 3" "262144 768 3" "65536 768 5"; do
    set -- $cfg
    INFCL_LIB=variants/libinfcl_prev3.so B=$1 D=$2 TAG="prev b=$1 d=$2" REPS=$3 python scripts/time_step.py
    B=$1 D=$2 TAG="r2.2 b=$1 d=$2" REPS=$3 python scripts/time_step.py
  done
done
