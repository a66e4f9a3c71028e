#!/bin/bash
# Round-2 final-tree sweep: throughput and peak memory vs global batch at n = 1 with the fused backward; one-step 4M at d = 768
mkdir -p gpurun_out
rm -f gpurun_out/sweep_b_r02j.jsonl
for cfg in "65536 512 20" "131072 512 8" "262144 512 4" "524288 512 3" "1048576 512 3" "65536 768 20" "262144 768 4" "1048576 768 3"; do
  set -- $cfg
  timeout 900 python bench.py --b $1 --d $2 --steps $3 --warmup 3 --no-cpu-baseline 2>>gpurun_out/sweep_b_r02j.err | tail -1 >> gpurun_out/sweep_b_r02j.jsonl
done
BS=4194304 timeout 1200 python scripts/big_b.py > gpurun_out/big_b_r02j.jsonl 2>&1; echo "big rc=$?"
python - <<'PY'
import json
for l in open('gpurun_out/sweep_b_r02j.jsonl'):
    try: d = json.loads(l)
    except Exception: continue
    print(d['config']['b'], d['config']['d'], round(d['value']), round(d['ms_per_step'], 2), round(d['fwd_ms'], 2), round(d['bwd_ms'], 2), d['peak_gb_per_gpu'], round(d['roofline']['frac'], 3), d['e2e']['value'] if d.get('e2e') else None)
PY
cat gpurun_out/big_b_r02j.jsonl | tail -2
