import sys, os, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2003_02989_b200 import distributed as D, workloads as wl, ops
from paper_2003_02989_b200.engine import ENGINE
for n in [int(x) for x in sys.argv[1:]]:
    c = wl.brickwork_circuit(n, 14, wl.SEED_BIG)
    obs = wl.z_sum(n)
    th = torch.zeros((1, 0), device="cuda")
    b = ENGINE.bind([c], [], [obs])
    e0 = float(b.execute(th)["expectations"][0, 0])
    bs = ENGINE.bind([c], [], [], want_state=True)
    st = bs.execute(th, want_state=True, want_expect=False)["state"]
    nrm = float((st.abs() ** 2).sum().double())
    # expectation from the state with torch
    idx = torch.arange(1 << n, device="cuda", dtype=torch.int64)
    p = (st[0].abs() ** 2).double()
    ez = 0.0
    for q in range(n):
        ez += float((p * (1 - 2 * ((idx >> q) & 1)).double()).sum())
    del st, p, idx
    ENGINE._bound.clear(); torch.cuda.empty_cache()
    e1, _ = D.run_sharded(c, obs, 1, D.LoopbackExchange(1))
    torch.cuda.empty_cache()
    print(n, "engine", e0, "from_state_torch", ez, "norm", nrm, "sharded_g1", e1, flush=True)
