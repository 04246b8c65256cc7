#!/bin/bash
set -u
mkdir -p gpurun_out/jit_r2p
python -c "import __graft_entry__ as E; E.build()" > /dev/null 2>&1
HS_JIT_DUMP=gpurun_out/jit_r2p timeout 300 python tools/quick_perf.py tf96 ws200 rn50f 2>&1 | grep cand/s
ls gpurun_out/jit_r2p | grep cubin
timeout 1500 python -m pytest -q -m gpu -x tests/test_gpu_block_classes.py tests/test_gpu_jit.py tests/test_gpu_heuristics.py tests/test_gpu_search_multi.py 2>&1 | tail -2
