#!/bin/bash
# three-role producer epilogue: which part bounds it? (A/B builds; exp1 no G math, exp2 no G staging, exp3 neither)
for r in 1 2; do
  INFCL_BWD3=1 TAG=three-role REPS=5 python scripts/time_step.py
  for e in 1 2 3; do INFCL_LIB=variants/libinfcl_exp$e.so INFCL_BWD3=1 TAG=exp$e REPS=5 python scripts/time_step.py; done
done
