#!/bin/bash
set -u
python -c "import __graft_entry__ as E; E.build()" > /dev/null 2>&1
timeout 900 python -m pytest -q -m gpu -x tests/test_gpu_splitting.py tests/test_gpu_modularity_split.py tests/test_gpu_dropin.py 2>&1 | tail -3
timeout 1500 python tools/split_probe.py 2>&1 | tail -12
