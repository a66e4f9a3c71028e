#!/bin/bash
# three-role producer epilogue: k of every 4 groups of G exponentials on the FMA pipe (A/B builds)
for r in 1 2; do
  INFCL_BWD3=1 TAG=three-role REPS=7 python scripts/time_step.py
  INFCL_LIB=variants/libinfcl_poly1.so INFCL_BWD3=1 TAG=poly1 REPS=7 python scripts/time_step.py
  INFCL_LIB=variants/libinfcl_poly2.so INFCL_BWD3=1 TAG=poly2 REPS=7 python scripts/time_step.py
  TAG=two-role REPS=7 python scripts/time_step.py
done
