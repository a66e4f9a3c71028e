#!/bin/bash
python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "grad_scale" 2>&1 | grep -E "assert|Error|passed|failed" | head -10
INFCL_DEBUG_WAITS=1 python scripts/time_step.py 2>&1 | grep -E "fwd_ms|FWD kernel|BWD kernel|role 1" | head -14
