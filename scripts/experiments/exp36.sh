#!/bin/bash
timeout 900 compute-sanitizer --tool racecheck --print-limit 200 python scripts/sanitize_step.py > gpurun_out/racecheck_full.log 2>&1
grep -E "Race reported|Write access|Read access" gpurun_out/racecheck_full.log | sed -E 's/\+0x[0-9a-f]+//' | sort | uniq -c | sort -rn | head -20
timeout 1800 python scripts/mutation_check.py
