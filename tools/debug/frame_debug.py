import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from circuits import random_circuit, random_observable
from oracle import qcflow_port as orc
from paper_2003_02989_b200 import ops, gates as G
from paper_2003_02989_b200.circuit import Circuit, ParamExpr, circuit_symbols
from paper_2003_02989_b200.engine import ENGINE
from paper_2003_02989_b200 import workloads as wl

def run(c, obs, theta, syms):
    res = {}
    for jit, frame in (("0", "0"), ("1", "0"), ("1", "1")):
        os.environ["QF_JIT"], os.environ["QF_FRAME"] = jit, frame
        ENGINE._bound.clear()
        res[(jit, frame)] = ops.expectation_and_gradient([c] * len(theta), syms, theta, obs)
    ref = np.array([orc.adjoint_grad(c, obs[0], dict(zip(syms, t.astype(np.float64))))[1] for t in theta])
    for k, (e, g) in res.items():
        print("  ", k, "grad err vs oracle", float(np.max(np.abs(g - ref))))

n = 11
cases = {
 "pair_X": Circuit(n, [G.h(q) for q in range(n)] + [G.rx(0.3, 1), wl.pauli_pair_pow("X", "s0", 1, 2), G.ry(0.2, 2)]),
 "pair_Z_after_rx_sym": Circuit(n, [G.h(q) for q in range(n)] + [G.rx(ParamExpr("s1"), 1), wl.pauli_pair_pow("X", "s0", 1, 2)]),
 "cnotpow_sym": Circuit(n, [G.h(q) for q in range(n)] + [G.rx(ParamExpr("s1"), 3), G.cnot_pow(ParamExpr("s0"), 3, 4), G.ry(ParamExpr("s1"), 4)]),
 "cnotpow_sym2": Circuit(n, [G.h(q) for q in range(n)] + [G.rx(ParamExpr("s1"), 4), G.cnot_pow(ParamExpr("s0"), 3, 4), G.ry(ParamExpr("s1"), 3)]),
}
rng = np.random.default_rng(3)
obs = [random_observable(rng, n, diag=True, k=6)]
for name, c in cases.items():
    syms = circuit_symbols(c)
    theta = rng.uniform(-3, 3, size=(2, len(syms))).astype(np.float32)
    print(name, syms)
    run(c, obs, theta, syms)
