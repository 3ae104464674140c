import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2003_02989_b200 import workloads as wl, ops as qops
from paper_2003_02989_b200.circuit import circuit_symbols
from paper_2003_02989_b200.engine import ENGINE
circ, cost = wl.qaoa_circuit(20, 4, wl.qaoa_graph(20))
syms = circuit_symbols(circ)
th = torch.as_tensor(wl.qaoa_params(256, 4)).cuda()
host = torch.as_tensor(wl.qaoa_params(256, 4)).pin_memory()
b = ENGINE.bind([circ] * 256, syms, [cost], want_grad=True)
def t(fn, k=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): fn()
    e1.record(); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / k, 2)
res = []
for it in range(3):
    res.append(("exec", t(lambda: b.execute(th, want_grad=True))))
    res.append(("e2e", t(lambda: qops.expectation_and_gradient([circ] * 256, syms, host, [cost]))))
    res.append(("exec_sync", t(lambda: (b.execute(th, want_grad=True), torch.cuda.synchronize()))))
print(os.environ.get("QF_CKPT_PAD", "0"), os.environ.get("QF_CKPT", "1"), res)
