import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
from test_distributed import mixed_circuit, obs_all
from dist_oracle import OracleExecutor
from paper_2003_02989_b200 import distributed as D, workloads as wl
from paper_2003_02989_b200.circuit import circuit_symbols

class Tap:
    def __init__(self, inner): self.inner, self.log = inner, []
    def zeros(self, r, d): return self.inner.zeros(r, d)
    def apply(self, circs, names, vals, psi, obs=None):
        psi, e = self.inner.apply(circs, names, vals, psi, obs)
        self.log.append((psi.detach().cpu().numpy().astype(np.complex128).copy(), None if e is None else e.detach().cpu().numpy()))
        return psi, e

for n, g in [(9, 1), (11, 1), (12, 2)]:
    c = mixed_circuit(n, 11 * n + g)
    obs = obs_all(n)
    syms = circuit_symbols(c)
    vals = np.linspace(-1.1, 1.7, len(syms)).astype(np.float32)
    te, to = Tap(D.EngineExecutor()), Tap(OracleExecutor())
    e1, p = D.run_sharded(c, obs, g, D.LoopbackExchange(g), te, syms, vals)
    e2, _ = D.run_sharded(c, obs, g, D.LoopbackExchange(g), to, syms, vals)
    print(n, g, "engine", e1, "oracle", e2, [s.kind for s in p.steps])
    for k, ((a, ea), (b, eb)) in enumerate(zip(te.log, to.log)):
        print("  step", k, "max|d|", float(np.max(np.abs(a - b))), ea, eb)
# plain rotation circuit through from_state engine vs oracle
from paper_2003_02989_b200.engine import ENGINE
from oracle import qcflow_port as orc
c = mixed_circuit(9, 5)
syms = circuit_symbols(c)
vals = np.linspace(-1.1, 1.7, len(syms)).astype(np.float32)
init = np.zeros(512, np.complex64); init[0] = 1
b = ENGINE.bind([c], syms, [], from_state=True, want_state=True)
st = b.execute(torch.as_tensor(vals[None]).cuda(), initial=torch.as_tensor(init[None]).cuda(), want_state=True, want_expect=False)["state"]
ref = orc.simulate_amps(c, dict(zip(syms, vals.astype(np.float64))))
print("from_state 9q max|d|", float(np.max(np.abs(st.cpu().numpy()[0] - ref))))
