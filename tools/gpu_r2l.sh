#!/bin/bash
set -u
mkdir -p gpurun_out/jit_r2l
python -c "import __graft_entry__ as E; E.build()" > /dev/null 2>&1
HS_JIT_DUMP=gpurun_out/jit_r2l timeout 300 python tools/quick_perf.py tf96 2>&1 | grep cand/s
ls gpurun_out/jit_r2l
OPTS='"" dsmem=0 tregs=24 near=4 tlanes=256 ahead=1' WL="tf96" bash tools/jit_sweep.sh
