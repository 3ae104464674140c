import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2003_02989_b200 import workloads as wl
from paper_2003_02989_b200.circuit import Circuit
from paper_2003_02989_b200.engine import ENGINE
n = int(sys.argv[1])
full = wl.brickwork_circuit(n, 14, wl.SEED_BIG)
th = torch.zeros((1, 0), device="cuda")
os.environ["QF_JIT"] = "1"
for k in [int(x) for x in sys.argv[2:]]:
    c = Circuit(n, full.gates[:k])
    ENGINE._bound.clear(); ENGINE._plans.clear()
    b = ENGINE.bind([c], [], [], want_state=True)
    st = b.execute(th, want_state=True, want_expect=False)["state"]
    v = (st.abs() ** 2).double()
    print(k, "norm", float(v.sum()), "passes", len(b.plan.fwd.prog.passes), flush=True)
    del st, v; torch.cuda.empty_cache()
