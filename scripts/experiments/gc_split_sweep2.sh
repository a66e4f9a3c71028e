#!/bin/bash
# fused backward consumer count at larger batches (d = 512: b = 262144; d = 768: b = 262144), medians of 3
for r in 1 2; do
  for c in 19 21 22 23 25; do INFCL_GC_CONSUMERS=$c B=262144 TAG="b262144 c=$c" REPS=3 python scripts/time_step.py; done
  for c in 23 25 27 29; do INFCL_GC_CONSUMERS=$c B=262144 D=768 TAG="b262144 d768 c=$c" REPS=3 python scripts/time_step.py; done
done
