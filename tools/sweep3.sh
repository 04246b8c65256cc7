#!/bin/bash
# Direct-load specialised kernel: occupancy / register-budget sweep (ws200)
# and parity of the direct path under the JIT tests.
mkdir -p gpurun_out
python -c "import __graft_entry__ as E; E.build()" > /dev/null 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
nvidia-smi --query-compute-apps=pid,name,used_memory --format=csv
export QP_N=${QP_N:-8388608}
for o in ${OPTS:-"" "genes=reg" "genes=reg,lanes=128,ctas=2" "genes=reg,lanes=128,ctas=3,near=8,regs=40" "genes=reg,lanes=128,ctas=3,near=8,regs=48" "genes=reg,lanes=96,ctas=4,near=8,regs=40" "genes=reg,lanes=64,ctas=6,near=8,regs=40" "genes=reg,lanes=128,ctas=4,near=8,regs=24" "genes=reg,lanes=64,ctas=8,near=8,regs=24" "genes=reg,lanes=256,ctas=1,near=8,regs=48"}; do
  echo "== $o"
  HS_JIT_OPTS=$o timeout 300 python tools/quick_perf.py ${WL:-ws200} 2>&1 | tail -${TAILN:-1}
done
for o in ${POPTS:-"genes=reg,lanes=128,ctas=3,near=8,regs=40"}; do
  echo "== parity $o"
  HS_JIT_OPTS=$o timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
done
