#!/bin/bash
python -c "
import ctypes; L=ctypes.CDLL('paper_2410_17243_b200/libinfcl.so')
for c in (1,2,4,8,16): print('cluster', c, 'max active clusters', L.infcl_diag_max_clusters(c), flush=True)
"
for P in 74 37 18; do TAG=pairs$P INFCL_PAIRS=$P python scripts/time_step.py; done
TAG=noepi_pairs74 INFCL_DEBUG_NOEPI=1 INFCL_DEBUG_WAITS=1 python scripts/time_step.py 2>&1 | grep -v dbg
TAG=noepi_pairs37 INFCL_PAIRS=37 INFCL_DEBUG_NOEPI=1 INFCL_DEBUG_WAITS=1 python scripts/time_step.py 2>&1 | grep -v dbg
