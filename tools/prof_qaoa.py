"""Small QAOA 20q forward+adjoint run for ncu profiling (B=32)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2003_02989_b200 import workloads as wl
from paper_2003_02989_b200.circuit import circuit_symbols
from paper_2003_02989_b200.engine import ENGINE
B = int(os.environ.get("QF_B", "32"))
circ, cost = wl.qaoa_circuit(20, 4, wl.qaoa_graph(20))
syms = circuit_symbols(circ)
theta = torch.as_tensor(wl.qaoa_params(B, 4)).cuda()
b = ENGINE.bind([circ] * B, syms, [cost], want_grad=True)
for _ in range(2):
    out = b.execute(theta, want_grad=True)
torch.cuda.synchronize()
print("ok", out["expectations"][0].item())
