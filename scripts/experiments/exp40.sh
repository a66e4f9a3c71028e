#!/bin/bash
# sanitizers + CUDA mutation check after the resident-A forward and diagonal-term init
mkdir -p gpurun_out
bash scripts/sanitize.sh > gpurun_out/e40_sanitize.log 2>&1
timeout 1500 python scripts/mutation_check.py > gpurun_out/e40_mutation.log 2>&1; echo "rc=$?" >> gpurun_out/e40_mutation.log
