#!/bin/bash
# fused backward at cfg2: library default consumer count vs 22 / 23 (interleaved, medians of 7)
for r in 1 2 3 4; do
  TAG=default REPS=7 python scripts/time_step.py
  INFCL_GC_CONSUMERS=22 TAG=c22 REPS=7 python scripts/time_step.py
  INFCL_GC_CONSUMERS=23 TAG=c23 REPS=7 python scripts/time_step.py
done
INFCL_DEBUG_WAITS=1 TAG=dbg REPS=1 python scripts/time_step.py 2>&1 | grep "consumers\|P_c\|producers" | head -3
