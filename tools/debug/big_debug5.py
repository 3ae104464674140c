import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2003_02989_b200 import workloads as wl
from paper_2003_02989_b200.circuit import Circuit
from paper_2003_02989_b200.engine import ENGINE
n = int(sys.argv[1]); k = int(sys.argv[2])
full = wl.brickwork_circuit(n, 14, wl.SEED_BIG)
c = Circuit(n, full.gates[:k])
th = torch.zeros((1, 0), device="cuda")
res = {}
for jit in ("0", "1"):
    os.environ["QF_JIT"] = jit
    ENGINE._bound.clear(); ENGINE._plans.clear()
    b = ENGINE.bind([c], [], [], want_state=True)
    for p in range(1, len(b.plan.fwd.prog.passes) + 1):
        pass
    st = b.execute(th, want_state=True, want_expect=False)["state"]
    res[jit] = st.clone(); del st
d = (res["0"] - res["1"]).abs()[0]
bad = torch.nonzero(d > 1e-4).reshape(-1)
print("n", n, "k", k, "bad", bad.numel(), "of", d.numel())
if bad.numel():
    b64 = bad.to(torch.int64)
    ones = [int(((b64 >> q) & 1).sum()) for q in range(n)]
    print("bit-set counts among bad:", ones)
    print("first bad", bad[:8].tolist(), "jit vals", res["1"][0, bad[:4]].tolist(), "ref", res["0"][0, bad[:4]].tolist())
