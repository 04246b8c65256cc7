#!/bin/bash
# Option sweep of the specialised evaluator (quick_perf, ws200) + parity of
# the new code-generation paths under the JIT tests.
mkdir -p gpurun_out
python -c "import __graft_entry__ as E; E.build()" > /dev/null 2>&1
export QP_N=${QP_N:-8388608}
for o in "" "lanes=128" "lanes=192" "genes=reg" "near=8,regs=32" "genes=reg,near=8,regs=32" "genes=reg,near=8,regs=48" "genes=reg,near=16,regs=32" "genes=reg,avail=reg" "max=int" "genes=reg,near=8,regs=32,lanes=192"; do
  echo "== $o"
  HS_JIT_OPTS=$o timeout 300 python tools/quick_perf.py ${WL:-ws200} 2>&1 | tail -${TAILN:-1}
done
for o in "genes=reg" "genes=reg,near=8,regs=32"; do
  echo "== parity $o"
  HS_JIT_OPTS=$o timeout 600 python -m pytest tests/test_gpu_jit.py -x -q 2>&1 | tail -2
done
echo "== bench vs probe"
timeout 300 python bench.py --no-cpu --no-tts --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['roofline']['kernel_ms'], d['clocks'])"
timeout 300 python bench.py --no-cpu --no-tts --steps 40 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['roofline']['kernel_ms'], d['clocks'])"
QP_N=16777216 timeout 300 python tools/quick_perf.py ws200
