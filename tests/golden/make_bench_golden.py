"""Golden circuits of the reference's benchmark families (qcflow/bench.py:53-86), generated
with the real reference in the build container:

    python tests/golden/make_bench_golden.py   ->  tests/golden/bench_families.json

Each case stores the reference circuit (qcflow JSON schema) for (family, n, depth, seed)
and its simulated amplitudes (complex128, re/im lists); the GPU box reads only the JSON."""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from qcflow.bench import gen_random_dense, gen_structured  # noqa: E402
from qcflow.circuit import to_json  # noqa: E402
from qcflow.rng import derive_seed  # noqa: E402
from qcflow.sim import simulate  # noqa: E402

cases = []
for family, n, depth, i in [("random_dense", 6, 3, 0), ("random_dense", 7, 4, 1), ("structured", 8, 3, 0)]:
    seed = derive_seed(0, n, i)
    c = gen_random_dense(n, depth, seed) if family == "random_dense" else gen_structured(n, depth, 4, seed)
    a = simulate(c).amplitudes
    cases.append({"family": family, "n": n, "depth": depth, "index": i, "seed": int(seed),
                  "circuit": to_json(c), "re": a.real.tolist(), "im": a.imag.tolist()})
with open(os.path.join(HERE, "bench_families.json"), "w") as f:
    json.dump(cases, f)
print("wrote", len(cases), "cases")
