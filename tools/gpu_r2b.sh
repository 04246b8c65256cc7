#!/bin/bash
# Round-2 session b: new GPU tests, ncu capture of the bench kernel (full
# set + launch list), specialised-kernel SASS dump, compute-sanitizer.
set -u
mkdir -p gpurun_out/jit
T=${TAG:-r2b}
python -c "import __graft_entry__ as E; E.build()" > gpurun_out/${T}_build.log 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest -q -m gpu -x -rs tests/test_gpu_validate.py tests/test_gpu_nccl.py \
  tests/test_gpu_throughput_mode.py tests/test_gpu_dropin.py > gpurun_out/${T}_pytest_new.log 2>&1
echo "pytest new rc=$?"; tail -15 gpurun_out/${T}_pytest_new.log
HS_JIT_DUMP=gpurun_out/jit timeout 300 python tools/quick_perf.py ws200 ws1000 > gpurun_out/${T}_qp.log 2>&1; echo "qp rc=$?"; tail -4 gpurun_out/${T}_qp.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hs_jit_eval -s 3 -c 1 \
  -o gpurun_out/${T}_bench python bench.py --steps 3 --warmup 3 --no-cpu --no-tts --no-others > gpurun_out/${T}_ncu_full.log 2>&1
echo "ncu full rc=$?"
ncu -i gpurun_out/${T}_bench.ncu-rep --page raw --csv > gpurun_out/${T}_bench_raw.csv 2>/dev/null
ncu -i gpurun_out/${T}_bench.ncu-rep --page details --csv > gpurun_out/${T}_bench_details.csv 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-tts --no-others > /dev/null 2>&1
echo "ncu list rc=$?"
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_run.py jit trace search aot batched bounds validate \
    > gpurun_out/${T}_sanitize_${tool}.log 2>&1
  echo "sanitize $tool rc=$?"; tail -3 gpurun_out/${T}_sanitize_${tool}.log
done
