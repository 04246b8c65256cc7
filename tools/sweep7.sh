#!/bin/bash
python -c "import __graft_entry__ as E; E.build()" > /dev/null 2>&1
export QP_N=${QP_N:-8388608}
for o in "" "dur=sel" "near=12" "near=6" "near=12,regs=56" "fma=1,near=12" "ahead=3,near=12"; do
  echo "== $o"
  HS_JIT_OPTS=$o timeout 300 python tools/quick_perf.py ws200 rn50f 2>&1 | grep cand
done
