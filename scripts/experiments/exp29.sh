#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -x -q -k "e2e or paired_multi or narrow or cfg2" 2>&1 | tail -3
INFCL_FWD_NARROW=1 timeout 600 python -m pytest tests/test_gpu_large.py -x -q -k "e2e_host_entry_chunked" 2>&1 | tail -2
timeout 600 python bench.py --steps 20 > gpurun_out/bench_e2e2.json 2> gpurun_out/bench_e2e2.err; tail -1 gpurun_out/bench_e2e2.err
