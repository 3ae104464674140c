import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
os.environ["QF_JIT"] = "1"
from paper_2003_02989_b200 import workloads as wl, ops
from paper_2003_02989_b200.circuit import Circuit, circuit_symbols
from paper_2003_02989_b200.pauli import PauliString, PauliSum
from paper_2003_02989_b200.engine import ENGINE
for n in (16, 8, 4):
    phis, _, params = wl.qcnn_data(2, n)
    model = wl.qcnn_model(n)
    circs = [Circuit(n, list(wl.qcnn_data_circuit(p).gates) + list(model.gates)) for p in phis]
    syms = circuit_symbols(model)
    params = params[:, :len(syms)]
    obs = PauliSum([PauliString(1.0, {n - 1: "Z"})])
    res = {}
    for flag in ("1", "0"):
        os.environ["QF_BLOCK_ADJ"] = flag
        ENGINE._bound.clear()
        e, g = ops.expectation_and_gradient(circs, syms, params, [obs])
        res[flag] = np.asarray(g)
    d = np.abs(res["1"] - res["0"]).max(axis=0)
    bad = [(syms[i], round(float(d[i]), 5)) for i in np.argsort(-d)[:4] if d[i] > 1e-4]
    print(n, "max", float(d.max()), bad)
