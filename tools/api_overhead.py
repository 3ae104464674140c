"""Host overhead of the public API on the headline workload: wall time per call of
ops.expectation_and_gradient (pinned host rows -> numpy results) vs the bound graph replay
alone, and a cProfile of the API call (where the per-call microseconds go)."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2003_02989_b200 import ops, workloads as wl  # noqa: E402
from paper_2003_02989_b200.circuit import circuit_symbols  # noqa: E402
from paper_2003_02989_b200.engine import ENGINE  # noqa: E402

circ, cost = wl.qaoa_circuit(20, 4, wl.qaoa_graph(20))
syms = circuit_symbols(circ)
th = torch.as_tensor(wl.qaoa_params(256, 4)).pin_memory()
thd = th.cuda()
b = ENGINE.bind([circ] * 256, syms, [cost], want_grad=True)
for _ in range(3):
    ops.expectation_and_gradient([circ] * 256, syms, th, [cost])
    b.execute(thd, want_grad=True)
torch.cuda.synchronize()
N = 30
t0 = time.perf_counter()
for _ in range(N):
    out = b.execute(thd, want_grad=True)
    out["grad"].cpu()
torch.cuda.synchronize()
t_dev = (time.perf_counter() - t0) / N
t0 = time.perf_counter()
for _ in range(N):
    ops.expectation_and_gradient([circ] * 256, syms, th, [cost])
t_api = (time.perf_counter() - t0) / N
print(f"replay+sync {1e3 * t_dev:.3f} ms, public API {1e3 * t_api:.3f} ms, overhead {1e6 * (t_api - t_dev):.0f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    ops.expectation_and_gradient([circ] * 256, syms, th, [cost])
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
