#!/bin/bash
INFCL_LIB=variants/libinfcl_spin.so python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for round in 1 2; do
  TAG=base REPS=9 python scripts/time_step.py
  INFCL_LIB=variants/libinfcl_spin.so TAG=spin REPS=9 python scripts/time_step.py
  INFCL_SBOX=1 TAG=base_sb1 REPS=9 python scripts/time_step.py
  INFCL_SBOX=1 INFCL_LIB=variants/libinfcl_spin.so TAG=spin_sb1 REPS=9 python scripts/time_step.py
done
D=768 TAG=base REPS=5 python scripts/time_step.py
D=768 INFCL_LIB=variants/libinfcl_spin.so TAG=spin REPS=5 python scripts/time_step.py
