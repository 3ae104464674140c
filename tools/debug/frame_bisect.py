import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from circuits import random_circuit, random_observable
from oracle import qcflow_port as orc
from paper_2003_02989_b200 import ops
from paper_2003_02989_b200.circuit import Circuit, circuit_symbols
from paper_2003_02989_b200.engine import ENGINE
os.environ["QF_JIT"] = "1"
rng = np.random.default_rng(303)
n = 12
full = random_circuit(rng, n, 200, n_sym=5)
obs = [random_observable(rng, n, diag=True, k=6)]
def err(k):
    c = Circuit(n, full.gates[:k])
    syms = circuit_symbols(c)
    if not syms: return 0.0
    th = np.linspace(-2, 2, 2 * len(syms)).reshape(2, -1).astype(np.float32)
    out = {}
    for fr in ("0", "1"):
        os.environ["QF_FRAME"] = fr; ENGINE._bound.clear()
        out[fr] = ops.expectation_and_gradient([c] * 2, syms, th, obs)[1]
    return float(np.max(np.abs(out["0"] - out["1"])))
lo, hi = 1, 200
print("full", err(200))
while hi - lo > 1:
    mid = (lo + hi) // 2
    if err(mid) > 1e-4: hi = mid
    else: lo = mid
print("first failing prefix", hi, "err", err(hi))
for j in range(max(0, hi - 6), hi):
    g = full.gates[j]
    print(j, g.targets, g.name, None if g.exponent is None else (g.exponent.symbol, g.exponent.coeff, g.exponent.const),
          None if g.generator is None else [(t.coefficient, dict(t.factors)) for t in g.generator.terms])
