#!/bin/bash
python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "grad_scale or e2e" 2>&1 | tail -2
INFCL_DEBUG_WAITS=1 python scripts/time_step.py 2>&1 | grep -E "fwd_ms|FWD kernel|BWD kernel|role 1" | head -14
INFCL_DEBUG_NOTMA=1 INFCL_DEBUG_NOEPI=1 INFCL_DEBUG_WAITS=1 python scripts/time_step.py 2>&1 | grep -E "FWD kernel|role 1" | head -6
