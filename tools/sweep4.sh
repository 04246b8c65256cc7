#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as E; E.build()" > /dev/null 2>&1
export QP_N=${QP_N:-8388608}
for o in "" "genes=reg" "genes=reg,ahead=1" "genes=reg,ahead=2" "genes=reg,ahead=4" "ahead=2" "genes=reg,ahead=2,lanes=128,ctas=2" "genes=reg,ahead=2,near=8,regs=48" "genes=reg,ahead=2,regs=80"; do
  echo "== $o"
  HS_JIT_OPTS=$o timeout 300 python tools/quick_perf.py ws200 2>&1 | tail -1
done
for o in "genes=reg,ahead=2" "ahead=2"; do
  echo "== parity $o"
  HS_JIT_OPTS=$o timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
done
