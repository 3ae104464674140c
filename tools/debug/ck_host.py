import os, sys, time, cProfile, pstats
sys.path.insert(0, os.getcwd())
import torch
from paper_2003_02989_b200 import workloads as wl, ops as qops
from paper_2003_02989_b200.circuit import circuit_symbols
from paper_2003_02989_b200.engine import ENGINE
circ, cost = wl.qaoa_circuit(20, 4, wl.qaoa_graph(20))
syms = circuit_symbols(circ)
host = torch.as_tensor(wl.qaoa_params(256, 4)).pin_memory()
for _ in range(3):
    qops.expectation_and_gradient([circ] * 256, syms, host, [cost])
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
for _ in range(5):
    qops.expectation_and_gradient([circ] * 256, syms, host, [cost])
pr.disable()
print("wall per call ms", (time.perf_counter() - t0) / 5 * 1e3)
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
