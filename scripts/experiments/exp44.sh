#!/bin/bash
# SM reservation for the ring transfer: pair kernel on 74 / 73 / 72 pairs, alone and beside a 1-GB copy
mkdir -p gpurun_out
for P in 74 73 72; do
  INFCL_PAIRS=$P timeout 200 python scripts/experiments/overlap_probe.py | sed "s/^/pairs=$P /"
done > gpurun_out/e44_overlap.log 2>&1
