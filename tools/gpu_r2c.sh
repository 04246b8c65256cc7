#!/bin/bash
# r2c: parity of the codegen changes (maxsel setp.and, grouped TMEM loads,
# constant-memory communication terms), multi-chain SA, perf sweep, synccheck probes.
set -u
mkdir -p gpurun_out
T=${TAG:-r2c}
python -c "import __graft_entry__ as E; E.build(); E.smoke()" > gpurun_out/${T}_build.log 2>&1; echo "build+smoke rc=$?"; tail -1 gpurun_out/${T}_build.log
timeout 1500 python -m pytest -q -m gpu -x -s tests/test_gpu_search_multi.py tests/test_gpu_jit.py tests/test_gpu_parity.py \
  tests/test_gpu_fullsize.py tests/test_gpu_heuristics.py > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?"; grep -E "chains|passed|failed|Error" gpurun_out/${T}_pytest.log | tail -8
for o in "" "tlanes=512,tregs=24" "tlanes=512,tregs=32" "tlanes=448,tregs=32" "tregs=48" "ahead=3" "near=12"; do
  echo "opts=[$o]"; HS_JIT_OPTS=$o timeout 300 python tools/quick_perf.py ws200 ws30 rn50f tf96 2>&1 | grep -E "cand/s" | sed 's/(.*best/best/; s/ blocks.*gen/ gen/'
done
timeout 600 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_run.py jit > gpurun_out/${T}_sync_jit.log 2>&1; echo "synccheck jit rc=$?"
HS_SEARCH_AOT=1 timeout 600 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_run.py search > gpurun_out/${T}_sync_search_aot.log 2>&1; echo "synccheck search aot rc=$?"
HS_JIT_SEARCH=1 timeout 600 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_run.py search > gpurun_out/${T}_sync_search_jit.log 2>&1; echo "synccheck search jit rc=$?"; grep -E "Barrier|at hs|ERROR SUMMARY" gpurun_out/${T}_sync_search_jit.log | head -5
timeout 600 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_run.py aot batched bounds validate > gpurun_out/${T}_sync_rest.log 2>&1; echo "synccheck rest rc=$?"
