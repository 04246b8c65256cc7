#!/bin/bash
# r2f: host-side packing (tests + e2e), SASS dump of the default kernel,
# full bench line.
set -u
mkdir -p gpurun_out/jit_r2f
T=${TAG:-r2f}
python -c "import __graft_entry__ as E; E.build(); E.smoke()" > gpurun_out/${T}_build.log 2>&1; echo "build+smoke rc=$?"; tail -1 gpurun_out/${T}_build.log
nproc; lscpu | grep -E "Model name|Socket|Thread|NUMA node\(s\)" 
timeout 900 python -m pytest -q -m gpu -x tests/test_gpu_host_pack.py tests/test_gpu_parity.py > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
HS_JIT_DUMP=gpurun_out/jit_r2f timeout 300 python tools/quick_perf.py ws200 2>&1 | grep cand/s
timeout 1200 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2f_bench.json').read().strip().splitlines()[-1])
print("value", d["value"], "frac", d["roofline"]["frac"], "issue", (d["roofline"].get("issue") or {}).get("frac"))
e=d["e2e"]; print("e2e", e["value"], e["h2d_bytes_per_step"], "no_pack", e["u8_without_host_packing"]["value"], "p3", e["packed3_genomes"]["value"], "p2", e["packed2_genomes"]["value"])
PY
tail -3 gpurun_out/${T}_bench.err
