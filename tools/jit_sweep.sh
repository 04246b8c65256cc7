#!/bin/bash
# A/B the specialised kernel's code-generation options on one GPU.
for o in ${OPTS:-"avail=smem,dur=smem,regs=64,win=400" "avail=smem,dur=smem,regs=64,win=400,max=int" "avail=smem,dur=smem,regs=32,win=96" "avail=smem,dur=smem,regs=96,win=400"}; do
  echo "== $o"
  HS_JIT_OPTS=$o timeout 300 python tools/quick_perf.py ${WL:-ws200 ws30 rn50f ws_stack_10x20} 2>&1 | grep -v specialize
done
