#!/bin/bash
# r2e: device column in TMEM slots (tdev) + gword sweep, full GPU suite,
# bench warm-up fix, synccheck of hs_jit_sa without a prior mbarrier kernel.
set -u
mkdir -p gpurun_out/jit_r2e
T=${TAG:-r2e}
python -c "import __graft_entry__ as E; E.build(); E.smoke()" > gpurun_out/${T}_build.log 2>&1; echo "build+smoke rc=$?"; tail -1 gpurun_out/${T}_build.log
OPTS='"" tdev=0 gword=1 tdev=1,gword=1' WL="ws200 ws30 rn50f tf96 ws_stack_10x20" bash tools/jit_sweep.sh
HS_JIT_DUMP=gpurun_out/jit_r2e timeout 300 python tools/quick_perf.py ws200 > /dev/null 2>&1
for k in 1 2; do timeout 600 python bench.py --no-cpu --no-tts --no-others > gpurun_out/${T}_bench_q$k.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/${T}_bench_q$k.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['roofline']['kernel_ms'], d['e2e']['value'], d['clocks'])"; done
timeout 600 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_run.py sa_only > gpurun_out/${T}_sync_sa_only.log 2>&1; echo "synccheck sa_only rc=$?"; grep -E "Barrier|ERROR SUMMARY" gpurun_out/${T}_sync_sa_only.log | head -3
timeout 2400 python -m pytest -q -m gpu tests > gpurun_out/${T}_pytest_all.log 2>&1
echo "pytest all rc=$?"; tail -3 gpurun_out/${T}_pytest_all.log
