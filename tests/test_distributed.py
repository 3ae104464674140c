"""Global-qubit sharding (distributed.py, BASELINE cfg 5 / SURVEY 8(e)): the schedule's
invariants, and sharded execution -- in one process (loopback exchange) and over a gloo
process group of 2 and 4 ranks -- against the unsharded oracle.  The per-rank compute here
is the oracle (tests/dist_oracle.py); the GPU runs of the same driver are in
tests/test_gpu_parity.py."""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from circuits import rotation_circuit
from dist_oracle import OracleExecutor
from oracle import qcflow_port as orc
from paper_2003_02989_b200 import distributed as D
from paper_2003_02989_b200 import gates as G
from paper_2003_02989_b200 import workloads as wl
from paper_2003_02989_b200.circuit import Circuit, ParamExpr, circuit_symbols
from paper_2003_02989_b200.pauli import PauliString, PauliSum

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def mixed_circuit(n, seed):
    """Brickwork plus symbolic rotations, symbolic ZZ (diagonal, may straddle global
    qubits), CZ / T / S and concrete diagonal gates on the top qubits."""
    rng = np.random.default_rng(seed)
    c = wl.brickwork_circuit(n, 4, seed)
    gs = list(c.gates)
    gs += list(rotation_circuit(rng, n, 40, n_sym=3).gates)
    for q in range(n - 1):
        gs.append(wl.pauli_pair_pow("Z", "s0", q, n - 1 - q) if q != n - 1 - q else G.t(q))
    gs += [G.cz(n - 1, n - 2), G.t(n - 1), G.s(n - 2), G.rz(0.3, n - 1), G.h(n - 1), G.rx(ParamExpr("s1", 0.7), n - 2)]
    return Circuit(n, gs)


def obs_all(n):
    terms = [PauliString(0.25)] + [PauliString(1.0 + 0.1 * q, {q: "Z"}) for q in range(n)]
    terms += [PauliString(0.5, {0: "X", n - 1: "Z"}), PauliString(-0.3, {1: "Y", n - 2: "Z", n - 1: "Z"})]
    return PauliSum(terms)


@pytest.mark.parametrize("n,g", [(8, 1), (9, 2), (10, 3), (12, 2)])
def test_plan_invariants(n, g):
    c = mixed_circuit(n, n + g)
    plan = D.plan_segments(c, g)
    seen = []
    for step, pos in zip(plan.steps, plan.pos_before):
        assert sorted(pos) == list(range(n))
        if step.kind != "segment":
            continue
        for j in step.gates:
            gt = c.gates[j]
            if not D._gate_is_diag(gt):
                assert all(pos[q] < plan.n_loc for q in gt.targets), (j, gt.targets)
        seen += step.gates
    assert sorted(seen) == list(range(len(c.gates)))
    # dependency order respected on every qubit (diagonal gates may reorder among themselves)
    order = {j: k for k, j in enumerate(seen)}
    last = {}
    for j, gt in enumerate(c.gates):
        for q in gt.targets:
            if q in last and not (D._gate_is_diag(gt) and D._gate_is_diag(c.gates[last[q]])):
                assert order[last[q]] < order[j]
            last[q] = j


def test_brickwork_32q_needs_one_swap():
    c = wl.brickwork_circuit(32, 14, wl.SEED_BIG)
    for g in (1, 2, 3):
        plan = D.plan_segments(c, g)
        assert plan.swaps == 1 and not any(s.kind == "permute" for s in plan.steps)


def _reference(c, obs, vals):
    syms = circuit_symbols(c)
    amps = orc.simulate_amps(c, dict(zip(syms, np.asarray(vals, dtype=np.float32).astype(np.float64))))
    return orc.expectation(amps, obs, c.num_qubits)


@pytest.mark.parametrize("n,g", [(8, 1), (9, 2), (10, 3)])
def test_loopback_sharded_matches_oracle(n, g):
    c = mixed_circuit(n, 7 * n + g)
    obs = obs_all(n)
    syms = circuit_symbols(c)
    vals = np.linspace(-1.3, 2.1, len(syms))
    got, plan = D.run_sharded(c, obs, g, D.LoopbackExchange(g), OracleExecutor(), syms, vals)
    assert got == pytest.approx(_reference(c, obs, vals), abs=1e-10)


def test_permute_local_bits_matches_index_map():
    import torch

    n_loc = 5
    psi = torch.arange(2 * 32, dtype=torch.float64).reshape(2, 32).to(torch.complex128)
    perm = [3, 1, 4, 0, 2]
    out = D.permute_local_bits(psi, perm, n_loc)
    for i in range(32):
        j = sum(((i >> a) & 1) << perm[a] for a in range(n_loc))
        assert out[1, j] == psi[1, i]


WORKER = r"""
import os, sys
sys.path.insert(0, {root!r}); sys.path.insert(0, os.path.join({root!r}, "tests"))
import numpy as np, torch.distributed as dist
from dist_oracle import OracleExecutor
from test_distributed import mixed_circuit, obs_all
from paper_2003_02989_b200 import distributed as D
from paper_2003_02989_b200.circuit import circuit_symbols
dist.init_process_group("gloo")
g = {g}
n = {n}
c = mixed_circuit(n, 3)
obs = obs_all(n)
syms = circuit_symbols(c)
vals = np.linspace(-0.7, 1.9, len(syms))
e, plan = D.run_sharded(c, obs, g, D.NcclExchange(g), OracleExecutor(), syms, vals)
if dist.get_rank() == 0:
    np.save(os.environ["QF_OUT"], np.array([e, plan.swaps]))
dist.destroy_process_group()
"""


@pytest.mark.parametrize("g", [1, 2])
def test_gloo_sharded_state_matches_oracle(tmp_path, g):
    n = 9
    script = tmp_path / "w.py"
    script.write_text(WORKER.format(root=ROOT, g=g, n=n))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, QF_OUT=str(tmp_path / "out.npy"), MASTER_ADDR="127.0.0.1", OMP_NUM_THREADS="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={1 << g}",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), str(script)],
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    e, swaps = np.load(tmp_path / "out.npy")
    c = mixed_circuit(n, 3)
    obs = obs_all(n)
    syms = circuit_symbols(c)
    assert swaps >= 1
    assert e == pytest.approx(_reference(c, obs, np.linspace(-0.7, 1.9, len(syms))), abs=1e-10)


@pytest.mark.parametrize("n_loc,g", [(6, 1), (7, 2), (8, 3)])
def test_fused_swap_addressing_equals_all_to_all(n_loc, g):
    """The remote-store pass (jit.generate(remote_pass=...)) sends local amplitude idx of
    rank s to rank idx >> (n-g) at (idx & low) | (s << (n-g)); that is exactly the
    all-to-all the exchanges perform (LoopbackExchange.swap)."""
    import torch

    from paper_2003_02989_b200 import jit, planner as pl

    R = 1 << g
    psi = torch.arange(R << n_loc, dtype=torch.float64).reshape(R, -1).to(torch.complex128)
    want = D.LoopbackExchange(g).swap(psi.clone(), n_loc)
    got = torch.zeros_like(psi)
    SH, low = n_loc - g, (1 << (n_loc - g)) - 1
    for s in range(R):
        for idx in range(1 << n_loc):
            got[idx >> SH, (idx & low) | (s << SH)] = psi[s, idx]
    assert torch.equal(got, want)
    # and the generated kernel uses that formula
    c = wl.brickwork_circuit(12, 2, 1)
    prog = pl.build_program(c, pl.analyse(c, {}), 12, adjoint=False)
    src, names, _ = jit.generate(prog, "f", remote_pass=len(prog.passes) - 1, remote_g=2)
    assert names == [f"qf_f_p{len(prog.passes) - 1}_rs"]
    assert "a.peers[idx >> 10][(size_t)((idx & 1023u) | (myr << 10))]" in src[0]
