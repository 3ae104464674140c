import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
os.environ["QF_JIT"] = "1"
from paper_2003_02989_b200 import workloads as wl, ops
from paper_2003_02989_b200.circuit import Circuit, circuit_symbols
from paper_2003_02989_b200.pauli import PauliString, PauliSum
from paper_2003_02989_b200.engine import ENGINE
from oracle import qcflow_port as orc
n = 4
phis, _, params = wl.qcnn_data(2, n)
model = wl.qcnn_model(n)
circs = [Circuit(n, list(wl.qcnn_data_circuit(p).gates) + list(model.gates)) for p in phis]
syms = circuit_symbols(model)
params = params[:, :len(syms)]
obs = PauliSum([PauliString(1.0, {n - 1: "Z"})])
_, gg = orc.adjoint_grad(circs[0], obs, dict(zip(syms, params[0].astype(np.float64))))
print("oracle c0_6", gg[6])
for blk in ("1", "0"):
    for fr in ("1", "0"):
        for ck in ("1", "0"):
            os.environ.update(QF_BLOCK_ADJ=blk, QF_FRAME=fr, QF_CKPT=ck)
            ENGINE._bound.clear(); ENGINE._plans.clear()
            e, g = ops.expectation_and_gradient(circs, syms, params, [obs])
            b = ENGINE.bind(circs, syms, [obs], want_grad=True)
            print(blk, fr, ck, "frame", b.frame, "blocks", b.plan.adj.n_blocks, "ckpt", b.plan.extra.get("ckpt"),
                  "c0_6", float(np.asarray(g)[0, 6]), "maxerr", float(np.abs(np.asarray(g)[0] - gg).max()))
