#!/bin/bash
# host e2e entry: hybrid backward (fused over I rows [0, 10/16 b) + two-pass pieces) vs the two passes; parity first
timeout 900 python -m pytest tests/test_gpu_large.py -q -k "e2e" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "e2e" 2>&1 | tail -1
for r in 1 2 3; do
  INFCL_E2E_HYBRID=0 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('two-pass', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],3))"
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('hybrid  ', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],3))"
done
