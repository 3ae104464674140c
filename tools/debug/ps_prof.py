import os, sys, time, cProfile, pstats
sys.path.insert(0, os.getcwd())
import torch
from paper_2003_02989_b200 import workloads as wl, ops
from paper_2003_02989_b200.circuit import circuit_symbols
circ = wl.hea_circuit(10, 4); syms = circuit_symbols(circ)
th = torch.as_tensor(wl.hea_params(1024)).cuda(); obs = [wl.z_sum(10)]
for _ in range(2): ops.expectation_and_ps_gradient([circ] * 1024, syms, th, obs)
torch.cuda.synchronize()
pr = cProfile.Profile(); t0 = time.perf_counter(); pr.enable()
ops.expectation_and_ps_gradient([circ] * 1024, syms, th, obs); torch.cuda.synchronize()
pr.disable(); print("wall ms", (time.perf_counter() - t0) * 1e3)
pstats.Stats(pr).sort_stats("cumtime").print_stats(18)
