#!/bin/bash
# r2g: full GPU suite + bench line on the current tree.
set -u
mkdir -p gpurun_out
T=${TAG:-r2g}
python -c "import __graft_entry__ as E; E.build(); E.smoke()" > gpurun_out/${T}_build.log 2>&1; echo "build+smoke rc=$?"; tail -1 gpurun_out/${T}_build.log
timeout 2400 python -m pytest -q -m gpu tests -rs > gpurun_out/${T}_pytest_all.log 2>&1
echo "pytest all rc=$?"; tail -4 gpurun_out/${T}_pytest_all.log
timeout 1200 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err; echo "bench ref rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2g_bench.json').read().strip().splitlines()[-1])
r=json.loads(open('gpurun_out/r2g_bench_ref.json').read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"]["value"], "ref", r["value"], "ratio", d["value"]/r["value"], "e2e ratio", d["e2e"]["value"]/r["value"], "same config", d["config"]==r["config"])
print("split", json.dumps(d["split"])[:600])
PY
