#!/bin/bash
TAG=base python scripts/time_step.py
TAG=dbg INFCL_DEBUG_WAITS=1 python scripts/time_step.py 2>&1 | grep -v "infcl dbg"
TAG=noepi INFCL_DEBUG_NOEPI=1 INFCL_DEBUG_WAITS=1 python scripts/time_step.py 2>&1 | grep -E "tag|FWD|role [01]" | head -8
TAG=stages3 INFCL_STAGES=3 python scripts/time_step.py
