#!/bin/bash
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as E; E.build()" > /dev/null 2>&1
timeout 900 python -m pytest -q -m gpu -x tests/test_gpu_splitting.py tests/test_gpu_modularity_split.py 2>&1 | tail -2
timeout 1500 python tools/split_probe.py 2>&1 | tail -12
