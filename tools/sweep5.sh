#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as E; E.build()" > /dev/null 2>&1
export QP_N=${QP_N:-8388608}
for o in "ahead=2" "ahead=1" "ahead=3" "ahead=2,regs=48" "ahead=2,regs=80" "ahead=2,near=8,regs=48" "ahead=2,near=8,regs=64" "ahead=2,near=16,regs=56" "ahead=2,max=int" "ahead=3,regs=56"; do
  echo "== $o"
  HS_JIT_OPTS=$o timeout 300 python tools/quick_perf.py ws200 2>&1 | tail -1
done
for o in "" "ahead=2" "ahead=3"; do
  echo "== others $o"
  HS_JIT_OPTS=$o timeout 600 python tools/quick_perf.py ws30 rn50f iv3f tf96 ws_stack_10x20 2>&1 | grep cand
done
