#!/bin/bash
# fused backward G ring depth around P_c + 2 (cfg2: P_c = 22; b = 262144: P_c = 24 at ratio 2.2), medians
for r in 1 2 3; do
  for R in 22 24 26 30; do INFCL_GC_RING=$R TAG="ring=$R" REPS=7 python scripts/time_step.py; done
done
for r in 1 2; do
  for R in 24 26 28; do INFCL_GC_RING=$R B=262144 TAG="b262144 ring=$R" REPS=3 python scripts/time_step.py; done
  for R in 25 27 29 33; do INFCL_GC_RING=$R B=65536 D=768 TAG="d768 ring=$R" REPS=5 python scripts/time_step.py; done
done
