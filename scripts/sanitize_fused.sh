#!/bin/bash
mkdir -p gpurun_out
for tool in memcheck synccheck initcheck; do
  echo "== $tool"; timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_fused.py 2>&1 | tail -6
  echo "== $tool (three-role)"; INFCL_BWD3=1 timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_fused.py 2>&1 | tail -6
done
