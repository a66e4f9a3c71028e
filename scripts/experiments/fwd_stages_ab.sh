#!/bin/bash
# wide forward ring depth at cfg2 (resident A, 16-KB B stages) and d = 768 (streamed A, 32-KB stages), medians
for r in 1 2 3; do
  for ns in 4 5 6; do INFCL_STAGES=$ns TAG="fwd ns=$ns" REPS=7 python scripts/time_step.py; done
done
for r in 1 2; do
  for ns in 4 5 6; do INFCL_STAGES=$ns D=768 TAG="d768 fwd ns=$ns" REPS=5 python scripts/time_step.py; done
done
