import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2003_02989_b200 import workloads as wl, ops as qops
from paper_2003_02989_b200.circuit import circuit_symbols
from paper_2003_02989_b200.engine import ENGINE
circ, cost = wl.qaoa_circuit(20, 4, wl.qaoa_graph(20))
syms = circuit_symbols(circ)
th = torch.as_tensor(wl.qaoa_params(256, 4)).cuda()
b = ENGINE.bind([circ] * 256, syms, [cost], want_grad=True)
def t(fn, k=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k
print("execute", t(lambda: b.execute(th, want_grad=True)))
t0 = time.perf_counter(); [torch.cuda.mem_get_info(0) for _ in range(100)]; print("mem_get_info ms", (time.perf_counter() - t0) * 10)
x = [torch.empty((256, 1 << 20), dtype=torch.complex64, device="cuda") for _ in range(6)]
print("execute with 12GB held", t(lambda: b.execute(th, want_grad=True)))
host = torch.as_tensor(wl.qaoa_params(256, 4)).pin_memory()
print("e2e", t(lambda: qops.expectation_and_gradient([circ] * 256, syms, host, [cost])))
print("execute again", t(lambda: b.execute(th, want_grad=True)))
print(torch.cuda.memory_stats()["num_alloc_retries"], torch.cuda.memory_stats()["num_device_alloc"])
