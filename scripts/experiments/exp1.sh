#!/bin/bash
for D in 512 768; do
 TAG=base D=$D python scripts/time_step.py
 TAG=noepi D=$D INFCL_DEBUG_NOEPI=1 INFCL_DEBUG_WAITS=1 python scripts/time_step.py 2>&1 | grep -v "infcl dbg\]   role [23]"
 for S in 3 4 5; do TAG=stages$S D=$D INFCL_STAGES=$S python scripts/time_step.py; done
done
