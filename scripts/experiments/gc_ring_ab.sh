#!/bin/bash
# fused backward G ring depth (steps in flight; default P_c + 12 = 34 at cfg2) at cfg2 and b = 262144, medians
for r in 1 2 3; do
  for R in 24 34 46; do INFCL_GC_RING=$R TAG="ring=$R" REPS=7 python scripts/time_step.py; done
done
for r in 1 2; do
  for R in 25 35 47; do INFCL_GC_RING=$R B=262144 TAG="b262144 ring=$R" REPS=3 python scripts/time_step.py; done
done
