#!/bin/bash
# One GPU session: build, smoke, GPU tests, bench, ncu launch list + full
# capture of the evaluator. Outputs land in gpurun_out/ (merged back).
set -u
mkdir -p gpurun_out
TAG=${TAG:-s}
python -c "import __graft_entry__ as E; E.build(); E.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
tail -2 gpurun_out/${TAG}_smoke.log
if [ "${TESTS:-1}" = "1" ]; then
  timeout 900 python -m pytest tests -q -m gpu -x ${PYTEST_ARGS:-} > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
  tail -5 gpurun_out/${TAG}_pytest.log
fi
if [ "${BENCH:-1}" = "1" ]; then
  timeout 600 python bench.py ${BENCH_ARGS:-} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
  tail -c 3000 gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
fi
if [ "${NCU:-1}" = "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
     --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --n 4194304 --no-cpu --no-tts --no-others --e2e-n 1048576 > /dev/null 2>&1; echo "ncu list rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_K:-eval} -s 3 -c 1 \
     -o gpurun_out/${TAG}_eval python tools/quick_perf.py ${NCU_WL:-ws200} > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu full rc=$?"
  tail -3 gpurun_out/${TAG}_ncu.log
fi
