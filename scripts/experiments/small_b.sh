#!/bin/bash
for b in 8192 16384 32768 65536; do
  B=$b REPS=9 TAG=b$b python scripts/time_step.py
done
