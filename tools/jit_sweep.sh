#!/bin/bash
# A/B sweep of the specialised evaluator's code-generation options on one
# GPU (quick_perf: device throughput of explicit genomes, median of blocks).
#   OPTS="'' tlanes=512,tregs=24 ahead=3" WL="ws200 ws30" bash tools/jit_sweep.sh
# Options are HS_JIT_OPTS keys (csrc/jit.cpp JitOpts::from_env); "" is the
# default configuration. PARITY=1 re-runs the JIT parity tests per option.
eval "set -- ${OPTS:-\"\" tlanes=512,tregs=24 tregs=48 ahead=3 near=12}"
for o in "$@"; do
  echo "== opts=[$o]"
  HS_JIT_OPTS=$o timeout 600 python tools/quick_perf.py ${WL:-ws200 ws30 rn50f tf96 ws_stack_10x20} 2>&1 | grep "cand/s"
  if [ "${PARITY:-0}" = "1" ]; then
    HS_JIT_OPTS=$o timeout 900 python -m pytest tests/test_gpu_jit.py -x -q 2>&1 | tail -1
  fi
done
