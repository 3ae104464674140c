import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2003_02989_b200 import workloads as wl, gates as G
from paper_2003_02989_b200.circuit import Circuit
from paper_2003_02989_b200.engine import ENGINE

def norm_of(c, jit):
    os.environ["QF_JIT"] = jit
    ENGINE._bound.clear(); ENGINE._plans.clear()
    b = ENGINE.bind([c], [], [], want_state=True)
    st = b.execute(torch.zeros((1, 0), device="cuda"), want_state=True, want_expect=False)["state"]
    v = (st.abs() ** 2).double()
    r = float(v.sum()), float(v[0, : v.shape[1] // 2].sum())
    del st, v; torch.cuda.empty_cache()
    return r, len(b.plan.fwd.prog.passes)

n = int(sys.argv[1])
cases = {
  "h_all": Circuit(n, [G.h(q) for q in range(n)]),
  "h_all_rx_top": Circuit(n, [G.h(q) for q in range(n)] + [G.rx(0.3, n - 1), G.rx(0.2, 0)]),
  "rx_top_only": Circuit(n, [G.rx(0.3, n - 1), G.rx(0.4, n - 2)]),
  "cz_chain": Circuit(n, [G.h(q) for q in range(n)] + [G.cz(q, q + 1) for q in range(n - 1)] + [G.h(q) for q in range(n)]),
  "brick2": wl.brickwork_circuit(n, 2, 5),
}
for k, c in cases.items():
    for jit in ("1", "0"):
        print(n, k, "jit", jit, norm_of(c, jit), flush=True)
