#!/bin/bash
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_step.py 2>&1 | tail -8
done
