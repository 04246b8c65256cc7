#!/bin/bash
set -u
python -c "import __graft_entry__ as E; E.build()" > /dev/null 2>&1
timeout 1500 python -m pytest -q -m gpu -x tests/test_gpu_block_classes.py tests/test_gpu_jit.py tests/test_gpu_parity.py tests/test_gpu_search_multi.py 2>&1 | tail -3
OPTS='"" blk=0' WL="tf96" bash tools/jit_sweep.sh
timeout 300 python - <<'PY'
import json, time, sys
sys.path.insert(0, '.')
import paper_2308_00127_b200 as hs
g, hw, t = hs.load_instance(json.load(open('tests/golden/instances/tf96.json')))
hs.specialize(g, hw, t, 1)
for algo, fn in (("sa", hs.simulated_annealing), ("ea", hs.one_plus_one_ea)):
    fn(g, hw, t, 1, seed=0, budget=2000)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); s = fn(g, hw, t, 1, seed=0, budget=2000); ts.append(time.perf_counter() - t0)
    print(algo, "tf96", sorted(ts)[2] * 1e3, "ms", s.objective)
PY
