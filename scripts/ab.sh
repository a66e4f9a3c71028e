#!/bin/bash
# A/B timing of library variants (variants/libinfcl_*.so + the in-tree library), interleaved rounds
VARS=${VARS:-"prev new"}
for round in 1 2 3; do
  for v in $VARS; do
    if [ "$v" = new ]; then L=""; else L=variants/libinfcl_$v.so; fi
    INFCL_LIB=$L TAG=$v REPS=${REPS:-9} D=${D:-512} python scripts/time_step.py
  done
done
