import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2003_02989_b200 import workloads as wl, ops as qops
from paper_2003_02989_b200.circuit import circuit_symbols
from paper_2003_02989_b200.engine import ENGINE
circ, cost = wl.qaoa_circuit(20, 4, wl.qaoa_graph(20)); syms = circuit_symbols(circ)
th = torch.as_tensor(wl.qaoa_params(256, 4)).cuda()
host = torch.as_tensor(wl.qaoa_params(256, 4)).pin_memory()
b = ENGINE.bind([circ] * 256, syms, [cost], want_grad=True)
res = []
for i in range(80):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if (i // 10) % 2:
        qops.expectation_and_gradient([circ] * 256, syms, host, [cost])
    else:
        b.execute(th, want_grad=True)
    e1.record(); torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1))
r = np.array(res[2:])
st = torch.cuda.memory_stats()
print({k: os.environ.get(k) for k in ("QF_CKPT", "QF_CKPT_NOMEM", "QF_CKPT_CACHE")}, "median %.2f p90 %.2f max %.2f" % (np.median(r), np.percentile(r, 90), r.max()),
      "allocs", st["num_device_alloc"], "frees", st["num_device_free"], "retries", st["num_alloc_retries"])
