#!/bin/bash
# One GPU session on a gpurun box (outputs under gpurun_out/, merged back):
#
#   TAG=r2x STEPS="build tests bench ref ncu sanitize" bash tools/gpu_session.sh
#
# steps (in this order when listed):
#   build     build() + smoke()
#   tests     pytest -m gpu (PYTEST_ARGS to narrow it)
#   bench     python bench.py ${BENCH_ARGS}          -> ${TAG}_bench.json
#   ref       python bench.py --impl reference       -> ${TAG}_bench_ref.json
#   ncu       ncu --set full of the bench's own hs_jit_eval launch (+ raw /
#             details CSV, tools/ncu_summary.py) and the launch list of the
#             bench command (--metrics gpu__time_duration.sum)
#   sanitize  (refused on the current GPU pool since round 2's r4g: runs
#             under compute-sanitizer had left GPUs needing a reset; use
#             `python tools/sanitize_run.py` alone for its oracle checks)
#             compute-sanitizer memcheck / racecheck / synccheck over
#             tools/sanitize_run.py (synccheck of hs_jit_sa in its own
#             process: profiles/README.md r2c)
#   sweep     tools/jit_sweep.sh (OPTS, WL)
#   split     tools/split_probe.py
set -u
mkdir -p gpurun_out
T=${TAG:-s}
STEPS=${STEPS:-"build tests bench"}
has() { [[ " $STEPS " == *" $1 "* ]]; }
if has build; then
  python -c "import __graft_entry__ as E; E.build(); E.smoke()" > gpurun_out/${T}_build.log 2>&1
  echo "build+smoke rc=$?"; tail -1 gpurun_out/${T}_build.log
fi
if has tests; then
  timeout 2400 python -m pytest tests -q -m gpu -rs ${PYTEST_ARGS:-} > gpurun_out/${T}_pytest.log 2>&1
  echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
fi
if has bench; then
  timeout 1500 python bench.py ${BENCH_ARGS:-} > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
  echo "bench rc=$?"; tail -c 400 gpurun_out/${T}_bench.json; echo
fi
if has ref; then
  timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
  echo "ref rc=$?"; tail -c 300 gpurun_out/${T}_bench_ref.json; echo
fi
if has ncu; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:hs_jit_eval -s 3 -c 1 \
    -o gpurun_out/${T}_bench python bench.py --steps 3 --warmup 3 --no-cpu --no-tts --no-others \
    > gpurun_out/${T}_ncu_full.log 2>&1
  echo "ncu full rc=$?"
  ncu -i gpurun_out/${T}_bench.ncu-rep --page raw --csv > gpurun_out/${T}_bench_raw.csv 2>/dev/null
  ncu -i gpurun_out/${T}_bench.ncu-rep --page details --csv > gpurun_out/${T}_bench_details.csv 2>/dev/null
  python tools/ncu_summary.py gpurun_out/${T}_bench_raw.csv 16777216 > gpurun_out/${T}_bench_kernel_ncu.json
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-tts --no-others > /dev/null 2>&1
  echo "ncu list rc=$?"
fi
if has sanitize; then
  for tool in memcheck racecheck; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_run.py \
      > gpurun_out/${T}_sanitize_${tool}.log 2>&1
    echo "sanitize $tool rc=$?"
  done
  timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_run.py jit trace aot batched batched_jit gen bounds validate \
    > gpurun_out/${T}_sanitize_synccheck.log 2>&1; echo "synccheck rc=$?"
  timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_run.py sa_only \
    > gpurun_out/${T}_sanitize_synccheck_sa.log 2>&1; echo "synccheck sa rc=$?"
fi
if has sweep; then
  bash tools/jit_sweep.sh 2>&1 | tee gpurun_out/${T}_sweep.log
fi
if has split; then
  timeout 1500 python tools/split_probe.py 2>&1 | tee gpurun_out/${T}_split.log
fi
