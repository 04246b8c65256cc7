#!/bin/bash
# A/B the specialised kernel's code-generation options on one GPU.
for o in ${OPTS:-"regs=64,win=400" "lanes=320,regs=56,win=400" "lanes=320,regs=48,win=400" "lanes=288,regs=56,win=400"}; do
  echo "== $o"
  HS_JIT_OPTS=$o timeout 600 python tools/quick_perf.py ${WL:-ws200 ws30 rn50f tf96 ws_stack_10x20} 2>&1
done
