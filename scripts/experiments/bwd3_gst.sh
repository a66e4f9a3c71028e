#!/bin/bash
# three-role producers storing G with st.global (no staging smem; variant gst) with resident A (more B stages)
export INFCL_BWD3=1
INFCL_LIB=variants/libinfcl_gst.so INFCL_BWD3_RESA=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -k three_role 2>&1 | tail -1
INFCL_LIB=variants/libinfcl_gst.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -k three_role 2>&1 | tail -1
for r in 1 2; do
  INFCL_BWD3=0 TAG=two-role REPS=5 python scripts/time_step.py
  TAG=three-role REPS=5 python scripts/time_step.py
  INFCL_LIB=variants/libinfcl_gst.so TAG=gst-streamedA REPS=5 python scripts/time_step.py
  INFCL_LIB=variants/libinfcl_gst.so INFCL_BWD3_RESA=1 TAG=gst-residentA REPS=5 python scripts/time_step.py
done
INFCL_LIB=variants/libinfcl_gst.so INFCL_BWD3_RESA=1 INFCL_DEBUG_WAITS=1 TAG=dbg REPS=2 python scripts/time_step.py 2>&1 | grep -A30 "bwd3:" | grep -v "^{" | head -30
