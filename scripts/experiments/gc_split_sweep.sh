#!/bin/bash
# fused backward: consumer pair count sweep at cfg2 (d = 512) and b = 65536, d = 768 (medians of 5, interleaved)
for r in 1 2 3; do
  for c in 19 20 21 22 23 24; do INFCL_GC_CONSUMERS=$c TAG="c=$c" REPS=5 python scripts/time_step.py; done
done
for r in 1 2; do
  for c in 21 23 25 27; do INFCL_GC_CONSUMERS=$c D=768 TAG="d768 c=$c" REPS=5 python scripts/time_step.py; done
done
