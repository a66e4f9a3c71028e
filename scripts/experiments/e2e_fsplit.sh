#!/bin/bash
# host e2e hybrid backward: the fused part's share (sixteenths of b), interleaved
for r in 1 2 3; do
  for f in ${FS:-8 10 12}; do
    INFCL_E2E_FSPLIT=$f python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('f=$f', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],3))"
  done
done
