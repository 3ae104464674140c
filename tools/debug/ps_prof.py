import sys, os, time, cProfile, pstats
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
from paper_2003_02989_b200 import ops, workloads as wl
from paper_2003_02989_b200.circuit import circuit_symbols
circ = wl.hea_circuit(10, 4); syms = circuit_symbols(circ)
th = torch.as_tensor(wl.hea_params(1024)).cuda(); obs = [wl.z_sum(10)]
ops.expectation_and_ps_gradient([circ] * 1024, syms, th, obs); torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
t = time.time(); ops.expectation_and_ps_gradient([circ] * 1024, syms, th, obs); torch.cuda.synchronize(); print("wall", time.time() - t)
pr.disable(); pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
