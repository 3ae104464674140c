"""Ad-hoc GPU diagnostics: engine vs CPU oracle on small cases (prints errors)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from paper_2003_02989_b200 import workloads as wl, gates as G
from paper_2003_02989_b200.engine import ENGINE
from paper_2003_02989_b200.circuit import circuit_symbols, Circuit, ParamExpr
from paper_2003_02989_b200.pauli import PauliSum, PauliString
from oracle import qcflow_port as orc

def rand_circ(rng, n, depth, nsym):
    F1 = [G.x, G.y, G.z, G.h, G.s, G.t]; P1 = [G.rx, G.ry, G.rz, G.xpow, G.ypow, G.zpow]; F2 = [G.cz, G.cnot, G.swap]
    gs = []; names = [f"s{i}" for i in range(nsym)]
    for _ in range(depth):
        if rng.random() < 0.35:
            a, b = (int(q) for q in rng.choice(n, 2, replace=False)); r = rng.random()
            if r < 0.2: gs.append(G.cnot_pow(float(rng.uniform(-1.5,1.5)), a, b))
            elif r < 0.35: gs.append(G.cnot_pow(ParamExpr(names[rng.integers(nsym)], float(rng.uniform(-1.5,1.5)), float(rng.uniform(-.5,.5))), a, b))
            elif r < 0.5: gs.append(wl.pauli_pair_pow("XYZ"[rng.integers(3)], names[rng.integers(nsym)], a, b))
            else: gs.append(F2[rng.integers(3)](a, b))
        else:
            q = int(rng.integers(n)); r = rng.random()
            if r < 0.3: gs.append(F1[rng.integers(6)](q))
            elif r < 0.5: gs.append(P1[rng.integers(6)](float(rng.uniform(-2,2)), q))
            else: gs.append(P1[rng.integers(6)](ParamExpr(names[rng.integers(nsym)], float(rng.uniform(-1.5,1.5)), float(rng.uniform(-.5,.5))), q))
    return Circuit(n, gs)

rng = np.random.default_rng(5)
for trial in range(8):
    n = [6, 10, 13, 14, 15, 16, 17, 12][trial]
    circ = rand_circ(rng, n, 120, 5)
    syms = circuit_symbols(circ)
    theta = rng.uniform(-3, 3, size=(3, len(syms))).astype(np.float32)
    obs_d = PauliSum([PauliString(float(rng.uniform(-2,2)), {int(q): "Z" for q in rng.choice(n, size=int(rng.integers(1,3)), replace=False)}) for _ in range(4)])
    obs_g = PauliSum([PauliString(float(rng.uniform(-2,2)), {int(q): "XYZ"[rng.integers(3)] for q in rng.choice(n, size=int(rng.integers(1,3)), replace=False)}) for _ in range(4)])
    for obs in (obs_d, obs_g):
        out = ENGINE.run([circ]*3, syms, theta, [obs], want_state=True)
        st = out["state"].cpu().numpy(); E = out["expectations"].cpu().numpy()
        outg = ENGINE.run([circ]*3, syms, theta, [obs], want_grad=True)
        Gd = outg["grad"].cpu().numpy()
        es, ee, eg = 0, 0, 0
        for b in range(3):
            bind = dict(zip(syms, theta[b].astype(np.float64)))
            ref = orc.simulate_amps(circ, bind)
            e, g = orc.adjoint_grad(circ, obs, bind)
            es = max(es, np.abs(st[b] - ref).max()); ee = max(ee, abs(E[b,0]-e)); eg = max(eg, np.abs(Gd[b]-g).max())
        print(f"n={n} passes={out['plan'].fwd.prog.stats['passes']} state_err={es:.2e} E_err={ee:.2e} grad_err={eg:.2e}", flush=True)

# QAOA 20q timing
n=20; edges = wl.qaoa_graph(n); circ, cost = wl.qaoa_circuit(n, 4, edges); theta = wl.qaoa_params(256, 4)
syms = circuit_symbols(circ)
print(out['plan'].fwd.prog.stats)
for it in range(3):
    pass
for it in range(3):
    torch.cuda.synchronize(); t=time.time()
    out = ENGINE.run(circ, syms, torch.as_tensor(theta).cuda(), [cost], want_grad=True)
    torch.cuda.synchronize(); print("qaoa20 b256 value+grad", time.time()-t, flush=True)
print(ENGINE.run(circ, syms, torch.as_tensor(theta).cuda(), [cost], want_grad=True)['plan'].fwd.prog.stats)
bind = dict(zip(syms, theta[0].astype(np.float64)))
e, g = orc.adjoint_grad(circ, cost, bind)
print("row0 E", out["expectations"][0,0].item(), out['energy'][0].item(), e, "grad err", np.abs(out['grad'][0].cpu().numpy()-g).max())

# sampler bit-exactness on identical states
from paper_2003_02989_b200 import sampling as smp
for n in (10, 12, 16):
    circ = rand_circ(rng, n, 60, 3); syms = circuit_symbols(circ)
    theta = rng.uniform(-3, 3, size=(4, len(syms))).astype(np.float32)
    out = ENGINE.run([circ]*4, syms, theta, [], want_state=True)
    psi = out["state"]
    seeds = [11, 12, 13, 14]
    idx, near = smp.sample_indices(psi.contiguous(), n, 500, [smp.philox_key(s) for s in seeds])
    idx = idx.cpu().numpy(); st = psi.cpu().numpy().astype(np.complex128)
    mism = 0
    for b in range(4):
        ref = orc.draw_indices(st[b], n, 500, orc.substream(seeds[b]))
        mism += int((ref != idx[b]).sum())
    print(f"sample n={n}: mismatches={mism} near={near.cpu().numpy().tolist()}", flush=True)
