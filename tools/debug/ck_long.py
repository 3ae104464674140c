import os, sys, subprocess, threading, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import torch
import numpy as np
from paper_2003_02989_b200 import workloads as wl, ops as qops
from paper_2003_02989_b200.circuit import circuit_symbols
from paper_2003_02989_b200.engine import ENGINE
circ, cost = wl.qaoa_circuit(20, 4, wl.qaoa_graph(20)); syms = circuit_symbols(circ)
th = torch.as_tensor(wl.qaoa_params(256, 4)).cuda()
host = torch.as_tensor(wl.qaoa_params(256, 4)).pin_memory()
b = ENGINE.bind([circ] * 256, syms, [cost], want_grad=True)
samples = []
stop = False
def smi():
    while not stop:
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,clocks_event_reasons.active",
                            "--format=csv,noheader,nounits"], capture_output=True, text=True)
        samples.append((time.perf_counter(), r.stdout.strip()))
        time.sleep(0.05)
th_ = threading.Thread(target=smi); th_.start()
res = []
for i in range(120):
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if (i // 20) % 2:
        qops.expectation_and_gradient([circ] * 256, syms, host, [cost])
    else:
        b.execute(th, want_grad=True)
    e1.record(); torch.cuda.synchronize()
    res.append((t0, round(e0.elapsed_time(e1), 2), round((time.perf_counter() - t0) * 1e3, 2)))
stop = True; th_.join()
print(os.environ.get("QF_CKPT", "1"), [r[1] for r in res])
print("wall", [r[2] for r in res])
slow = [r for r in res if r[1] > 16]
for r in slow[:6]:
    near = [s[1] for s in samples if abs(s[0] - r[0]) < 0.1]
    print("slow", r[1], near)
fast = [r for r in res if r[1] < 15][5:8]
for r in fast:
    print("fast", r[1], [s[1] for s in samples if abs(s[0] - r[0]) < 0.1])
