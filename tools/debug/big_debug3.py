import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2003_02989_b200 import distributed as D, workloads as wl
from paper_2003_02989_b200.engine import ENGINE
n = int(sys.argv[1])
c = wl.brickwork_circuit(n, 14, wl.SEED_BIG)
obs = wl.z_sum(n)
th = torch.zeros((1, 0), device="cuda")
for env in [("QF_JIT", "1"), ("QF_JIT", "0"), ("QF_GEOM_FWD", "13,5")]:
    os.environ[env[0]] = env[1]
    ENGINE._bound.clear(); ENGINE._plans.clear()
    b = ENGINE.bind([c], [], [], want_state=True)
    st = b.execute(th, want_state=True, want_expect=False)["state"]
    v = (st.abs() ** 2).double()
    print(env, "norm", float(v.sum()), "norm_lo_half", float(v[0, :v.shape[1] // 2].sum()), flush=True)
    del st, v; torch.cuda.empty_cache()
    os.environ.pop(env[0])
for g in (1, 2):
    ENGINE._bound.clear(); ENGINE._plans.clear(); torch.cuda.empty_cache()
    ex = D.LoopbackExchange(g)
    e, plan = D.run_sharded(c, D.PauliSum([D.PauliString(1.0)]), g, ex)
    print("sharded g", g, "norm", e, flush=True)
