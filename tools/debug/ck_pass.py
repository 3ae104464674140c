import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import torch
import pass_times as PT
from paper_2003_02989_b200 import workloads as wl, ops as qops
from paper_2003_02989_b200.circuit import circuit_symbols
b, th = PT.bound_for("cfg2")
host = torch.as_tensor(wl.qaoa_params(256, 4)).pin_memory()
circ, cost = wl.qaoa_circuit(20, 4, wl.qaoa_graph(20)); syms = circuit_symbols(circ)
for i in range(24):
    PT.REC.clear()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if i % 2:
        qops.expectation_and_gradient([circ] * 256, syms, host, [cost])
    else:
        b.execute(th, want_grad=True)
    e1.record()
    torch.cuda.synchronize()
    ts = [round(a.elapsed_time(c), 2) for _, _, a, c in PT.REC]
    print(i, round(e0.elapsed_time(e1), 2), round(sum(ts), 2), ts)
