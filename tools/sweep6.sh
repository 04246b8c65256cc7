#!/bin/bash
python -c "import __graft_entry__ as E; E.build()" > /dev/null 2>&1
export QP_N=${QP_N:-8388608}
for o in "" "fma=1" "fma=1,ahead=3" "fma=1,regs=56" "fma=1,near=12"; do
  echo "== $o"
  HS_JIT_OPTS=$o timeout 300 python tools/quick_perf.py ws200 2>&1 | tail -1
done
echo "== others fma=1"
HS_JIT_OPTS=fma=1 timeout 600 python tools/quick_perf.py ws30 rn50f iv3f tf96 ws_stack_10x20 2>&1 | grep cand
echo "== parity fma=1"
HS_JIT_OPTS=fma=1 timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
