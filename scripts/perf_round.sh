#!/bin/bash
# d = 768 fused consumer split, cfg3 batch at N = 1 (fused vs two-pass), virtual ring per-step cost (fused / two-pass)
mkdir -p gpurun_out
for v in "" "INFCL_GC_CONSUMERS=19" "INFCL_GC_CONSUMERS=23" "INFCL_GC_CONSUMERS=25" "INFCL_FUSED_BWD=0"; do
  env $v TAG="$v d768" D=768 REPS=5 timeout 120 python scripts/time_step.py 2>&1 | tail -1
done
for v in "" "INFCL_FUSED_BWD=0"; do
  env $v TAG="$v cfg3-batch" B=262144 D=768 REPS=2 timeout 300 python scripts/time_step.py 2>&1 | tail -1
done
echo "== vring fused"; timeout 600 python scripts/experiments/vring_time.py 2>&1 | tail -4
echo "== vring two-pass"; INFCL_FUSED_BWD=0 timeout 600 python scripts/experiments/vring_time.py 2>&1 | tail -4
echo "== vring cfg3 per-rank (b=262144 over 8)"; B=262144 D=768 timeout 900 python scripts/experiments/vring_time.py 2>&1 | tail -4
