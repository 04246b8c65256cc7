#!/bin/bash
python -c "import __graft_entry__ as E; E.build()" > /dev/null 2>&1
export QP_N=${QP_N:-8388608}
for o in "tmem=1,lanes=384,regs=24" "tmem=1,lanes=384,regs=16"; do
  echo "== parity $o"
  HS_JIT_OPTS=$o timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3
done
for o in "tmem=1,lanes=384,regs=24" "tmem=1,lanes=384,regs=32" "tmem=1,lanes=352,regs=32" "tmem=1,lanes=416,regs=20" "tmem=1,lanes=448,regs=16" "tmem=1,lanes=384,regs=24,near=12" "tmem=1,lanes=384,regs=24,ahead=3"; do
  echo "== $o"
  HS_JIT_OPTS=$o timeout 300 python tools/quick_perf.py ws200 rn50f ws30 tf96 ws_stack_10x20 2>&1 | grep -E "cand|rror" | tail -5
done
