#!/bin/bash
# r2d: device EA draw + multi-chain tests, synccheck of the JIT search after
# the mbarrier invalidation, ncu of the bench kernel (new codegen), WS1000
# sweep, full bench line.
set -u
mkdir -p gpurun_out
T=${TAG:-r2d}
python -c "import __graft_entry__ as E; E.build(); E.smoke()" > gpurun_out/${T}_build.log 2>&1; echo "build+smoke rc=$?"; tail -1 gpurun_out/${T}_build.log
timeout 1500 python -m pytest -q -m gpu -x -s tests/test_gpu_search_multi.py tests/test_gpu_heuristics.py tests/test_gpu_dropin.py \
  > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?"; grep -E "chains|passed|failed|Error|assert" gpurun_out/${T}_pytest.log | tail -12
HS_JIT_SEARCH=1 timeout 600 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_run.py jit search > gpurun_out/${T}_sync_search_jit.log 2>&1; echo "synccheck jit+search rc=$?"; grep -E "Barrier|at hs|ERROR SUMMARY" gpurun_out/${T}_sync_search_jit.log | head -5
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hs_jit_eval -s 3 -c 1 \
  -o gpurun_out/${T}_bench python bench.py --steps 3 --warmup 3 --no-cpu --no-tts --no-others > gpurun_out/${T}_ncu_full.log 2>&1
echo "ncu full rc=$?"
ncu -i gpurun_out/${T}_bench.ncu-rep --page raw --csv > gpurun_out/${T}_bench_raw.csv 2>/dev/null
ncu -i gpurun_out/${T}_bench.ncu-rep --page details --csv > gpurun_out/${T}_bench_details.csv 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-tts --no-others > /dev/null 2>&1
echo "ncu list rc=$?"
for o in "" "glanes=256" "glanes=320" "glanes=384" "sync=16" "ahead=0" "near=4"; do
  echo "ws1000 opts=[$o]"; HS_JIT_OPTS=$o QP_N=2097152 timeout 300 python tools/quick_perf.py ws1000 2>&1 | grep -E "cand/s" | sed 's/(.*best/best/; s/ blocks.*gen/ gen/'
done
timeout 1200 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2d_bench.json').read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"]["value"], "frac", d["roofline"]["frac"])
print(json.dumps(d.get("time_to_solution"))[:1500])
PY
