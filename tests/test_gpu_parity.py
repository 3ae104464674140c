"""GPU parity tests: the CUDA path (through the drop-in API / C ABI) vs the CPU oracle
and the reference's golden vectors.

Tolerances (BASELINE.json north star, complex64 arithmetic):
  * amplitudes             1e-5 absolute
  * expectations           1e-4 absolute
  * gradients              1e-4 absolute + 1e-5 relative.  The relative part only matters for
                           gradients above ~10 in magnitude: complex64 itself cannot do better
                           there (the same adjoint restated in NumPy complex64 is off by 1.7e-4 on
                           the 16-qubit QAOA family with |g| ~ 23).
  * sampled bitstrings     bit-exact for identical states and seeds.
"""

import json

import numpy as np
import pytest

from circuits import random_circuit, random_observable
from oracle import qcflow_port as orc
from paper_2003_02989_b200 import gates as G
from paper_2003_02989_b200 import gradients as gr
from paper_2003_02989_b200 import ops, sim
from paper_2003_02989_b200 import workloads as wl
from paper_2003_02989_b200.circuit import Circuit, ParamExpr, Symbol, circuit_symbols, from_json, resolve
from paper_2003_02989_b200.pauli import PauliString, PauliSum, identity, pauli_sum_from_obj, pauli_x, pauli_z

pytestmark = pytest.mark.gpu

AMP, EXP, GABS, GREL = 1e-5, 1e-4, 1e-4, 1e-5


def _obs(s):
    return pauli_sum_from_obj(json.loads(s))


def _close_grad(got, want):
    np.testing.assert_allclose(got, want, atol=GABS, rtol=GREL)


# ---------------------------------------------------------------------------
# golden vectors from the reference
# ---------------------------------------------------------------------------


def test_known_answers(cuda, golden):
    meta, arr = golden
    bell = from_json(meta["cases"]["bell"]["circuit"])
    s = sim.simulate(bell)
    np.testing.assert_allclose(s.amplitudes, arr["bell/amps"], atol=AMP)
    assert sim.expectation(s, PauliString(1.0, {0: "Z", 1: "Z"})) == pytest.approx(1.0, abs=EXP)
    assert sim.expectation(s, pauli_z(0)) == pytest.approx(0.0, abs=EXP)
    c = Circuit(1, [G.xpow(Symbol("theta"), 0)])
    out = sim.batch_execute([c, c, c], [[0.0], [1.0], [2.0]], [pauli_z(0)])
    np.testing.assert_allclose(out, [[1.0], [-1.0], [1.0]], atol=EXP)
    # little endian: X on qubit q sets bit q
    for q in range(6):
        st = sim.simulate(Circuit(6, [G.x(q)]))
        np.testing.assert_allclose(st.amplitudes, np.eye(64)[1 << q], atol=AMP)
        assert sim.expectation(st, pauli_z(q)) == pytest.approx(-1.0, abs=EXP)


@pytest.mark.parametrize("i", range(8))
def test_golden_states_and_expectations(cuda, golden, i):
    meta, arr = golden
    case = meta["cases"][f"concrete{i}"]
    c = from_json(case["circuit"])
    st = sim.simulate(c)
    np.testing.assert_allclose(st.amplitudes, arr[f"concrete{i}/amps"], atol=AMP)
    for o, e in zip(case["observables"], case["expectations"]):
        assert sim.expectation(st, _obs(o)) == pytest.approx(e, abs=EXP)


@pytest.mark.parametrize("i", range(4))
def test_golden_gradients_adjoint_and_ps(cuda, golden, i):
    meta, arr = golden
    case = meta["cases"][f"symbolic{i}"]
    c = from_json(case["circuit"])
    o = _obs(case["observable"])
    b = dict(zip(case["symbols"], case["bindings"]))
    req = gr.GradRequest(c, o, b)
    _close_grad(gr.adjoint_grad(req).gradient, arr[f"symbolic{i}/ps"])
    ps = gr.parameter_shift_grad(req)
    _close_grad(ps.gradient, arr[f"symbolic{i}/ps"])
    assert ps.evaluations == case["ps_evaluations"]


def test_golden_config_families(cuda, golden):
    meta, arr = golden
    cfg = meta["configs"]
    for name in ("hea", "qaoa"):
        c = from_json(cfg[name]["circuit"])
        o = _obs(cfg[name]["observable"])
        rows = np.array(cfg[name]["rows"], dtype=np.float32)
        e, g = ops.expectation_and_gradient(c, circuit_symbols(c), rows, [o])
        np.testing.assert_allclose(e, arr[f"{name}/exp"], atol=EXP)
        _close_grad(g, arr[f"{name}/ps"])
    c = from_json(cfg["qcnn"]["circuit"])
    o = _obs(cfg["qcnn"]["observable"])
    e, g = ops.expectation_and_gradient(c, circuit_symbols(c), np.array([cfg["qcnn"]["row"]], dtype=np.float32), [o])
    np.testing.assert_allclose(e[0], arr["qcnn/exp"][0], atol=EXP)
    _close_grad(g[0], arr["qcnn/ps"])
    c = from_json(cfg["rcs"]["circuit"])
    np.testing.assert_allclose(sim.simulate(c).amplitudes, arr["rcs/amps"], atol=AMP)
    c = from_json(cfg["big"]["circuit"])
    assert sim.expectation(sim.simulate(c), _obs(cfg["big"]["observable"])) == pytest.approx(
        cfg["big"]["expectation"], abs=EXP)


# ---------------------------------------------------------------------------
# CUDA path vs oracle on seeded random inputs
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("seed,n", [(0, 3), (1, 9), (2, 10), (3, 12), (4, 13), (5, 14), (6, 16), (7, 17)])
def test_states_expectations_gradients_vs_oracle(cuda, seed, n):
    rng = np.random.default_rng(100 + seed)
    c = random_circuit(rng, n, 150, n_sym=5)
    syms = circuit_symbols(c)
    theta = rng.uniform(-3, 3, size=(3, len(syms))).astype(np.float32)
    obs = [random_observable(rng, n, diag=True), random_observable(rng, n, diag=False)]
    states = ops.state([c] * 3, syms, theta)
    e, g = ops.expectation_and_gradient([c] * 3, syms, theta, obs, upstream=np.array([[1.0, 0.5]] * 3))
    for b in range(3):
        bind = dict(zip(syms, theta[b].astype(np.float64)))
        ref = orc.simulate_amps(c, bind)
        np.testing.assert_allclose(states[b], ref, atol=AMP)
        for k, o in enumerate(obs):
            assert e[b, k] == pytest.approx(orc.expectation(ref, o, n), abs=EXP)
        weighted = obs[0] + obs[1] * 0.5
        _close_grad(g[b], orc.adjoint_grad(c, weighted, bind)[1])


def test_batch_rows_with_different_concrete_values(cuda):
    """QCNN-style data circuits: same topology, per-row concrete angles (ref graph.py:443-468)."""
    rng = np.random.default_rng(7)
    model = wl.qcnn_model(8)
    rows = []
    for _ in range(5):
        data = wl.qcnn_data_circuit(rng.uniform(-np.pi, np.pi, 8))
        rows.append(Circuit(8, tuple(data.gates) + tuple(model.gates)))
    syms = circuit_symbols(model)
    theta = rng.uniform(0, 2, size=(5, len(syms))).astype(np.float32)
    z7 = PauliSum([PauliString(1.0, {7: "Z"})])
    e, g = ops.expectation_and_gradient(rows, syms, theta, [z7])
    for b in range(5):
        bind = dict(zip(syms, theta[b].astype(np.float64)))
        ee, gg = orc.adjoint_grad(rows[b], z7, bind)
        assert e[b, 0] == pytest.approx(ee, abs=EXP)
        _close_grad(g[b], gg)


def test_sampler_bit_exact_on_identical_states(cuda):
    import torch

    from paper_2003_02989_b200.sampling import philox_key, sample_indices

    rng = np.random.default_rng(11)
    for n in (10, 13, 16):
        c = random_circuit(rng, n, 80)
        psi = ops.state([c] * 3, [], torch.zeros((3, 0), device="cuda"))
        seeds = [3, 99, 123456]
        idx, near = sample_indices(psi.contiguous(), n, 700, [philox_key(s) for s in seeds])
        st = psi.cpu().numpy().astype(np.complex128)
        for b in range(3):
            want = orc.draw_indices(st[b], n, 700, orc.substream(seeds[b]))
            np.testing.assert_array_equal(idx[b].cpu().numpy(), want)
        assert int(near.sum()) == 0


def test_sample_api_matches_oracle_draw_on_gpu_state(cuda):
    rng = np.random.default_rng(12)
    c = random_circuit(rng, 7, 40)
    st = sim.simulate(c)
    got = sim.sample(st, 500, seed=17).bitstrings
    want = orc.sample(st.device_amplitudes().cpu().numpy().astype(np.complex128), 7, 500, 17)
    np.testing.assert_array_equal(got, want)
    with pytest.raises(ValueError):
        sim.sample(st, 0, seed=1)


def test_sampled_expectation_bit_exact_semantics(cuda):
    """Same draw semantics as ref sim.py:245-272: feed the oracle the GPU's rotated states."""
    rng = np.random.default_rng(13)
    c = random_circuit(rng, 5, 30)
    obs = PauliSum([PauliString(0.8, {0: "X", 2: "Z"}), PauliString(-0.5, {1: "Y"}), identity(0.25),
                    PauliString(0.3, {3: "Z", 4: "Z"})])
    got = sim.sampled_expectation(c, obs, 600, seed=101)
    rotated = {}
    for k, t in enumerate(obs.terms):
        if t.factors:
            rc = Circuit(5, tuple(c.gates) + tuple(sim.basis_change_gates(t)))
            rotated[k] = sim.simulate(rc).device_amplitudes().cpu().numpy().astype(np.complex128)
    want = orc.sampled_expectation(c, obs, 600, 101, rotated_states=rotated)
    assert got == pytest.approx(want, abs=1e-12)
    # exact cases (ref test_sim.py:284-306)
    bell = Circuit(2, [G.h(0), G.cnot(0, 1)])
    assert sim.sampled_expectation(bell, PauliString(1.0, {0: "Z", 1: "Z"}), 2000, seed=11) == 1.0
    assert sim.sampled_expectation(Circuit(1, [G.h(0)]), pauli_x(0), 2000, seed=13) == 1.0
    assert sim.sampled_expectation(Circuit(1, [G.h(0), G.s(0)]), PauliString(1.0, {0: "Y"}), 500, seed=17) == 1.0
    assert sim.sampled_expectation(Circuit(1, []), PauliSum([identity(2.5), pauli_z(0)]), 1, seed=0) == 3.5


def test_run_ops_apply_matrix_unitary(cuda):
    rng = np.random.default_rng(14)
    from circuits import random_unitary

    n = 5
    amps = rng.normal(size=(4, 2 ** n)) + 1j * rng.normal(size=(4, 2 ** n))
    amps /= np.linalg.norm(amps, axis=1, keepdims=True)
    for tg in [(0,), (2,), (4,), (1, 3), (3, 1), (0, 4), (4, 2)]:
        u = random_unitary(2 ** len(tg), rng)
        np.testing.assert_allclose(sim.apply_matrix(amps, u, tg, n), orc.apply_matrix(amps, u, tg, n), atol=AMP)
    c = random_circuit(rng, 3, 12)
    np.testing.assert_allclose(sim.unitary(c)[:, 0], sim.simulate(c).amplitudes, atol=AMP)


def test_parameter_shift_gpu_matches_oracle_ps(cuda):
    rng = np.random.default_rng(15)
    c = random_circuit(rng, 6, 40, n_sym=4)
    o = random_observable(rng, 6)
    b = {s: float(rng.uniform(-2, 2)) for s in circuit_symbols(c)}
    want, n_eval = orc.parameter_shift_grad(c, o, b)
    res = gr.parameter_shift_grad(gr.GradRequest(c, o, b))
    _close_grad(res.gradient, want)
    assert res.evaluations == n_eval
    fd = gr.finite_difference_grad(gr.GradRequest(c, o, b), epsilon=2e-3)
    np.testing.assert_allclose(fd.gradient, want, atol=5e-3)


# ---------------------------------------------------------------------------
# edge cases and error behaviour (reference exception classes)
# ---------------------------------------------------------------------------


def test_edge_cases(cuda, monkeypatch):
    st = sim.simulate(Circuit(3))
    np.testing.assert_allclose(st.amplitudes, np.eye(8)[0], atol=AMP)
    assert sim.expectation(sim.StateVector.zero(1), identity(2.5)) == 2.5
    with pytest.raises(KeyError, match="t"):
        sim.simulate(Circuit(1, [G.rx("t", 0)]))
    monkeypatch.setenv("QCFLOW_MAX_QUBITS", "3")
    with pytest.raises(MemoryError, match="QCFLOW_MAX_QUBITS"):
        sim.simulate(Circuit(4, [G.h(0)]))
    monkeypatch.setenv("QCFLOW_MAX_QUBITS", "junk")
    with pytest.raises(ValueError, match="junk"):
        sim.simulate(Circuit(4, [G.h(0)]))
    monkeypatch.delenv("QCFLOW_MAX_QUBITS")
    c = Circuit(2, [G.rx("a", 0), G.ry("b", 1)])
    with pytest.raises(ValueError, match="ragged"):
        sim.batch_execute([c], [[0.1]], [pauli_z(0)])
    assert sim.batch_execute([], [], [pauli_z(0)]).shape == (0, 1)
    with pytest.raises(ValueError, match="commute"):
        bad = Circuit(1, [G.Gate((0,), exponent=ParamExpr("s"), generator=PauliSum([pauli_x(0), pauli_z(0)]))])
        gr.parameter_shift_grad(gr.GradRequest(bad, pauli_z(0), {"s": 0.3}))
    with pytest.raises(KeyError):
        gr.adjoint_grad(gr.GradRequest(c, pauli_z(0), {"a": 0.1}))
    # zero upstream -> zero gradient; identity-only generator contributes zero
    _, g = ops.expectation_and_gradient(c, ["a", "b"], np.array([[0.3, 0.4]], np.float32), [pauli_z(0)],
                                        upstream=np.zeros((1, 1)))
    np.testing.assert_allclose(g, 0.0, atol=1e-12)


def test_batch_permutation_invariance_and_upstream_linearity(cuda):
    circ, cost = wl.qaoa_circuit(12, 2, wl.qaoa_graph(12, seed=5))
    syms = circuit_symbols(circ)
    th = wl.qaoa_params(6, 2)
    perm = np.array([3, 0, 5, 1, 4, 2])
    e1, g1 = ops.expectation_and_gradient(circ, syms, th, [cost])
    e2, g2 = ops.expectation_and_gradient(circ, syms, th[perm], [cost])
    np.testing.assert_allclose(e2, e1[perm], atol=1e-12)
    np.testing.assert_allclose(g2, g1[perm], atol=1e-12)
    _, g3 = ops.expectation_and_gradient(circ, syms, th, [cost], upstream=np.full((6, 1), 2.5))
    np.testing.assert_allclose(g3, 2.5 * g1, rtol=1e-5, atol=1e-5)


# ---------------------------------------------------------------------------
# full-size properties (BASELINE configs) -- size-independent checks
# ---------------------------------------------------------------------------


def test_qaoa20_full_batch_properties(cuda):
    import torch

    circ, cost = wl.qaoa_circuit(20, 4, wl.qaoa_graph(20))
    syms = circuit_symbols(circ)
    th = torch.as_tensor(wl.qaoa_params(256, 4)).cuda()
    st = ops.state(circ, syms, th[:8])
    norms = (st.abs() ** 2).sum(dim=1).double().cpu().numpy()
    np.testing.assert_allclose(norms, 1.0, atol=1e-5)
    e, g = ops.expectation_and_gradient(circ, syms, th, [cost])
    assert e.shape == (256, 1) and g.shape == (256, 8)
    # spot-check two rows against the oracle's adjoint restatement
    for b in (0, 255):
        bind = dict(zip(syms, th[b].double().cpu().numpy()))
        ee, gg = orc.adjoint_grad(circ, cost, bind)
        assert float(e[b, 0]) == pytest.approx(ee, abs=EXP)
        _close_grad(g[b].cpu().numpy(), gg)


def test_rcs24_sampling_bit_exact(cuda):
    """Config 4 circuits at full size: 24 qubits, depth 20; bitstrings identical to the
    reference draw on the same (upcast) state and seed."""
    circs = wl.rcs_circuits(2, 24, 20)
    from paper_2003_02989_b200.sampling import derive_seed

    seeds = [derive_seed(wl.SEED_RCS_SHOTS, b) for b in range(2)]
    bits = ops.sample(circs, [], np.zeros((2, 0), np.float32), 1000, seed=seeds)
    st = ops.state(circs, [], np.zeros((2, 0), np.float32))
    for b in range(2):
        want = orc.sample(st[b].astype(np.complex128), 24, 1000, seeds[b])
        np.testing.assert_array_equal(bits[b], want)
    norms = (np.abs(st) ** 2).sum(axis=1)
    np.testing.assert_allclose(norms, 1.0, atol=1e-5)


def test_plan_specialised_kernels_match_interpreter(cuda, monkeypatch):
    """The NVRTC-generated pass kernels (jit.py) and the interpreted pass kernel run the
    same programs; both must agree with the oracle (forward, adjoint, fused observables)."""
    rng = np.random.default_rng(21)
    c = random_circuit(rng, 15, 160, n_sym=5)
    syms = circuit_symbols(c)
    theta = rng.uniform(-3, 3, size=(4, len(syms))).astype(np.float32)
    obs = [random_observable(rng, 15, diag=True)]
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("QF_JIT", flag)
        from paper_2003_02989_b200.engine import ENGINE

        ENGINE._bound.clear()
        st = ops.state([c] * 4, syms, theta)
        e, g = ops.expectation_and_gradient([c] * 4, syms, theta, obs)
        out[flag] = (st, e, g)
    np.testing.assert_allclose(out["1"][0], out["0"][0], atol=1e-6)
    np.testing.assert_allclose(out["1"][1], out["0"][1], atol=1e-6)
    np.testing.assert_allclose(out["1"][2], out["0"][2], atol=1e-5, rtol=1e-6)
    bind = dict(zip(syms, theta[0].astype(np.float64)))
    ee, gg = orc.adjoint_grad(c, obs[0], bind)
    assert out["1"][1][0, 0] == pytest.approx(ee, abs=EXP)
    _close_grad(out["1"][2][0], gg)


@pytest.mark.parametrize("seed,n,family", [(0, 11, "rot"), (1, 13, "rot"), (2, 14, "rot"), (3, 12, "any"),
                                           (4, 13, "any")])
def test_pauli_frame_normalised_programs_vs_oracle(cuda, monkeypatch, seed, n, family):
    """Plan-specialised kernels with Pauli-frame normalised rotations (engine default for
    diagonal observables): expectations and adjoint gradients against the oracle, and
    identical to the same kernels without the frame (QF_FRAME=0)."""
    from circuits import rotation_circuit
    from paper_2003_02989_b200.engine import ENGINE

    rng = np.random.default_rng(300 + seed)
    c = rotation_circuit(rng, n, 220, n_sym=6) if family == "rot" else random_circuit(rng, n, 200, n_sym=5)
    syms = circuit_symbols(c)
    theta = rng.uniform(-3.5, 3.5, size=(4, len(syms))).astype(np.float32)
    obs = [random_observable(rng, n, diag=True, k=6), random_observable(rng, n, diag=True, k=3)]
    monkeypatch.setenv("QF_JIT", "1")
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("QF_FRAME", flag)
        ENGINE._bound.clear()
        b = ENGINE.bind([c] * 4, syms, obs, want_grad=True)
        assert b.frame == (flag == "1")
        out[flag] = ops.expectation_and_gradient([c] * 4, syms, theta, obs, upstream=np.array([[1.0, -0.7]] * 4))
    np.testing.assert_allclose(out["1"][0], out["0"][0], atol=2e-5)
    np.testing.assert_allclose(out["1"][1], out["0"][1], atol=5e-5, rtol=1e-5)
    e_only = ops.expectation([c] * 4, syms, theta, obs)
    np.testing.assert_allclose(e_only, out["0"][0], atol=2e-5)
    for b in range(4):
        bind = dict(zip(syms, theta[b].astype(np.float64)))
        ref = orc.simulate_amps(c, bind)
        for k, o in enumerate(obs):
            assert out["1"][0][b, k] == pytest.approx(orc.expectation(ref, o, n), abs=EXP)
        _close_grad(out["1"][1][b], orc.adjoint_grad(c, obs[0] + obs[1] * -0.7, bind)[1])


@pytest.mark.parametrize("seed,n", [(0, 12), (1, 14), (2, 13), (3, 15)])
def test_checkpointed_adjoint_vs_oracle(cuda, monkeypatch, seed, n):
    """Checkpointed adjoint sweep (engine.Bound._checkpoints): forward pass outputs kept, the
    backward passes reload psi from them.  Gradients and energies against the oracle and
    against the store-and-uncompute sweep (QF_CKPT=0); the plan must actually use it."""
    from circuits import pauli_rotation_circuit
    from paper_2003_02989_b200.engine import ENGINE

    rng = np.random.default_rng(700 + seed)
    c = pauli_rotation_circuit(rng, n, 240, n_sym=6)
    syms = circuit_symbols(c)
    theta = rng.uniform(-3.5, 3.5, size=(4, len(syms))).astype(np.float32)
    obs = [random_observable(rng, n, diag=True, k=6), random_observable(rng, n, diag=True, k=3)]
    monkeypatch.setenv("QF_JIT", "1")
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("QF_CKPT", flag)
        ENGINE._bound.clear()
        ENGINE._plans.clear()
        b = ENGINE.bind([c] * 4, syms, obs, want_grad=True)
        assert bool(b.plan.extra.get("ckpt")) == (flag == "1")
        out[flag] = ops.expectation_and_gradient([c] * 4, syms, theta, obs, upstream=np.array([[1.0, -0.7]] * 4))
    np.testing.assert_allclose(out["1"][0], out["0"][0], atol=2e-5)
    np.testing.assert_allclose(out["1"][1], out["0"][1], atol=5e-5, rtol=1e-5)
    for b in range(4):
        bind = dict(zip(syms, theta[b].astype(np.float64)))
        ref = orc.simulate_amps(c, bind)
        for k, o in enumerate(obs):
            assert out["1"][0][b, k] == pytest.approx(orc.expectation(ref, o, n), abs=EXP)
        _close_grad(out["1"][1][b], orc.adjoint_grad(c, obs[0] + obs[1] * -0.7, bind)[1])


@pytest.mark.parametrize("seed,n,diag", [(0, 9, True), (1, 12, True), (2, 11, False), (3, 13, True)])
def test_block_fused_adjoint_vs_oracle(cuda, monkeypatch, seed, n, diag):
    """Block-fused adjoint (planner.build_ops(block=True), qf_block_grads): symbolic gates
    fused into dense blocks, every factor's gradient from the block's two-point matrix.
    Against the oracle and against the per-gate sweep (QF_BLOCK_ADJ=0), with Pauli frames
    (diagonal observables) and without (an X/Y observable term)."""
    from paper_2003_02989_b200.engine import ENGINE

    rng = np.random.default_rng(900 + seed)
    c = random_circuit(rng, n, 260, n_sym=7, p2=0.45)
    syms = circuit_symbols(c)
    theta = rng.uniform(-2.5, 2.5, size=(4, len(syms))).astype(np.float32)
    obs = [random_observable(rng, n, diag=diag, k=5), random_observable(rng, n, diag=True, k=3)]
    monkeypatch.setenv("QF_JIT", "1")
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("QF_BLOCK_ADJ", flag)
        ENGINE._bound.clear()
        b = ENGINE.bind([c] * 4, syms, obs, want_grad=True)
        assert (b.plan.adj.n_blocks > 0) == (flag == "1")
        out[flag] = ops.expectation_and_gradient([c] * 4, syms, theta, obs, upstream=np.array([[0.8, -1.1]] * 4))
    np.testing.assert_allclose(out["1"][0], out["0"][0], atol=2e-5)
    np.testing.assert_allclose(out["1"][1], out["0"][1], atol=5e-5, rtol=1e-5)
    for b in range(4):
        bind = dict(zip(syms, theta[b].astype(np.float64)))
        _close_grad(out["1"][1][b], orc.adjoint_grad(c, obs[0] * 0.8 + obs[1] * -1.1, bind)[1])


# ---------------------------------------------------------------------------
# global-qubit sharding (distributed.py) on the engine
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("n,g", [(9, 1), (12, 2), (14, 3)])
def test_sharded_engine_matches_oracle(cuda, n, g):
    """The sharded schedule (loopback exchange: all 2^g shards on this GPU) with the CUDA
    engine per shard, against the unsharded oracle -- incl. diagonal gates and Z terms on
    global qubits and X/Y observable terms (a final swap makes their qubits local)."""
    from test_distributed import mixed_circuit, obs_all
    from paper_2003_02989_b200 import distributed as D

    c = mixed_circuit(n, 11 * n + g)
    obs = obs_all(n)
    syms = circuit_symbols(c)
    vals = np.linspace(-1.1, 1.7, len(syms)).astype(np.float32)
    got, plan = D.run_sharded(c, obs, g, D.LoopbackExchange(g), None, syms, vals)
    amps = orc.simulate_amps(c, dict(zip(syms, vals.astype(np.float64))))
    assert got == pytest.approx(orc.expectation(amps, obs, n), abs=EXP)


def test_sharded_brickwork_matches_unsharded_engine(cuda):
    """Config-5 family at 24 qubits: 1/2/3 global qubits give the single-GPU expectation."""
    from paper_2003_02989_b200 import distributed as D

    c = wl.brickwork_circuit(24, 14, wl.SEED_BIG)
    obs = wl.z_sum(24)
    want = float(ops.expectation(c, [], np.zeros((1, 0), np.float32), [obs])[0, 0])
    for g in (1, 2, 3):
        got, plan = D.run_sharded(c, obs, g, D.LoopbackExchange(g))
        assert plan.swaps == 1
        assert got == pytest.approx(want, abs=1e-5)


def test_large_register_30q_norm_and_sharding(cuda):
    """Index arithmetic above 2^29 amplitudes (8 GiB states): the norm is preserved and a
    2-shard run of the same circuit agrees with the single-GPU expectation."""
    import torch
    from paper_2003_02989_b200 import distributed as D

    n = 30
    c = wl.brickwork_circuit(n, 6, wl.SEED_BIG)
    st = ops.state(c, [], torch.zeros((1, 0), device="cuda"))
    assert float((st.abs() ** 2).double().sum()) == pytest.approx(1.0, abs=1e-4)
    del st
    torch.cuda.empty_cache()
    obs = wl.z_sum(n)
    want = float(ops.expectation(c, [], np.zeros((1, 0), np.float32), [obs])[0, 0])
    got, _ = D.run_sharded(c, obs, 1, D.LoopbackExchange(1))
    assert got == pytest.approx(want, abs=1e-5)
    torch.cuda.empty_cache()


def test_batched_parameter_shift_matches_reference_ps(cuda, golden):
    """ops.expectation_and_ps_gradient (all rows x shifts batched) against the reference's
    parameter-shift vectors (golden HEA config rows) and the oracle's PS on random rows."""
    meta, arr = golden
    cfg = meta["configs"]["hea"]
    c = from_json(cfg["circuit"])
    o = _obs(cfg["observable"])
    rows = np.array(cfg["rows"], dtype=np.float32)
    e, g = ops.expectation_and_ps_gradient(c, circuit_symbols(c), rows, [o])
    np.testing.assert_allclose(e, arr["hea/exp"], atol=EXP)
    _close_grad(g, arr["hea/ps"])
    rng = np.random.default_rng(44)
    c2 = random_circuit(rng, 6, 60, n_sym=4)
    syms = circuit_symbols(c2)
    th = rng.uniform(-2, 2, size=(3, len(syms))).astype(np.float32)
    o2 = random_observable(rng, 6)
    e2, g2 = ops.expectation_and_ps_gradient([c2] * 3, syms, th, [o2])
    for b in range(3):
        bind = dict(zip(syms, th[b].astype(np.float64)))
        _close_grad(g2[b], orc.parameter_shift_grad(c2, o2, bind)[0])


# ---------------------------------------------------------------------------
# determinism, re-entrancy and statistical bands (ref test_sim.py:250-334,
# test_bench_cli.py:206-214, test_gradients.py:275-325)
# ---------------------------------------------------------------------------


def test_concurrent_calls_are_deterministic(cuda):
    """The engine is re-entrant: calls from several threads give the serial results
    bit-for-bit (the reference's bench runs simulate from worker threads)."""
    from concurrent.futures import ThreadPoolExecutor

    rng = np.random.default_rng(71)
    c = random_circuit(rng, 12, 120, n_sym=4)
    syms = circuit_symbols(c)
    theta = rng.uniform(-2, 2, size=(6, len(syms))).astype(np.float32)
    obs = [random_observable(rng, 12, diag=True), random_observable(rng, 12)]
    want_e, want_g = ops.expectation_and_gradient([c] * 6, syms, theta, obs)
    want_s = sim.simulate(resolve(c, dict(zip(syms, theta[0].astype(np.float64))))).amplitudes

    def job(i):
        if i % 2:
            return ops.expectation_and_gradient([c] * 6, syms, theta, obs)
        return sim.simulate(resolve(c, dict(zip(syms, theta[0].astype(np.float64))))).amplitudes

    with ThreadPoolExecutor(4) as ex:
        outs = list(ex.map(job, range(8)))
    for i, o in enumerate(outs):
        if i % 2:
            np.testing.assert_array_equal(o[0], want_e)
            np.testing.assert_array_equal(o[1], want_g)
        else:
            np.testing.assert_array_equal(o, want_s)


def test_sampling_statistics_and_seed_determinism(cuda):
    c = Circuit(3, [G.h(0), G.x(2)])
    a = sim.sample(sim.simulate(c), 40000, seed=9)
    b = sim.sample(sim.simulate(c), 40000, seed=9)
    d = sim.sample(sim.simulate(c), 40000, seed=10)
    bits = np.asarray(a.bitstrings)
    np.testing.assert_array_equal(bits, np.asarray(b.bitstrings))
    assert not np.array_equal(bits, np.asarray(d.bitstrings))
    assert abs(bits[:, 0].mean() - 0.5) < 0.01          # binomial band (ref test_sim.py:259-271)
    assert bits[:, 1].sum() == 0 and bits[:, 2].min() == 1


def test_sampled_expectation_band_over_seeds(cuda):
    """Mean of sampled <Z0 + X1> over seeds within 5 sigma of the exact value (ref
    test_sim.py:318-334)."""
    c = Circuit(2, [G.ry(0.7, 0), G.rx(0.4, 1), G.h(1), G.cz(0, 1), G.h(1)])
    obs = PauliSum([PauliString(1.0, {0: "Z"}), PauliString(1.0, {1: "X"})])
    exact = sim.expectation(sim.simulate(c), obs)
    vals = np.array([sim.sampled_expectation(c, obs, 200, seed=s) for s in range(100)])
    sigma = np.sqrt(2.0 / 200 / 100)
    assert abs(vals.mean() - exact) < 5 * sigma


def test_fused_swap_pass_matches_all_to_all(cuda):
    """The global-qubit swap fused into the preceding pass (remote stores into the ranks'
    receive shards) gives the same sharded result as the separate all-to-all."""
    from paper_2003_02989_b200 import distributed as D

    c = wl.brickwork_circuit(22, 10, wl.SEED_BIG)
    obs = wl.z_sum(22)
    for g in (1, 2, 3):
        fused, plan = D.run_sharded(c, obs, g, D.LoopbackExchange(g), fuse_swaps=True)
        plain, _ = D.run_sharded(c, obs, g, D.LoopbackExchange(g), fuse_swaps=False)
        assert plan.swaps >= 1
        assert fused == pytest.approx(plain, abs=1e-6)


def test_qcnn16_plan_specialised_many_slot_passes(cuda, monkeypatch):
    """Config-3 QCNN at 16 qubits through the plan-specialised kernels: passes with more
    gradient slots than fit per thread use the 16-slot ring flushed by warp
    transpose-reductions; gradients against the oracle's adjoint."""
    from paper_2003_02989_b200.engine import ENGINE

    monkeypatch.setenv("QF_JIT", "1")
    ENGINE._bound.clear()
    phis, _, params = wl.qcnn_data(2, 16)
    model = wl.qcnn_model(16)
    circs = [Circuit(16, list(wl.qcnn_data_circuit(p).gates) + list(model.gates)) for p in phis]
    syms = circuit_symbols(model)
    obs = PauliSum([PauliString(1.0, {15: "Z"})])
    e, g = ops.expectation_and_gradient(circs, syms, params, [obs])
    b = ENGINE.bind(circs, syms, [obs], want_grad=True)
    assert max(int(p[9] - p[8]) for p in b.plan.adj.prog.passes) > 40     # ring mode exercised
    for r in range(2):
        bind = dict(zip(syms, params[r].astype(np.float64)))
        ee, gg = orc.adjoint_grad(circs[r], obs, bind)
        assert e[r, 0] == pytest.approx(ee, abs=EXP)
        _close_grad(g[r], gg)


# ---------------------------------------------------------------------------
# layer entry points (ref graph.py:443-549) with a PQC-shaped node
# ---------------------------------------------------------------------------


class _Node:
    """The attributes quantum_forward/backward use of the reference's _QuantumNode."""

    def __init__(self, model, data, observables, differentiator, estimator=None):
        self.name = "pqc"
        self.model_circuit = model
        self.symbols = circuit_symbols(model)
        self.observables = observables
        self.differentiator = differentiator
        self.estimator = estimator if estimator is not None else gr.Exact()
        self._data = data
        self._calls = 0

    def _data_batch(self, rows):
        return self._data[:rows]

    def _combined(self, d):
        return Circuit(self.model_circuit.num_qubits, list(d.gates) + list(self.model_circuit.gates))

    def _next_call(self):
        self._calls += 1
        return self._calls


@pytest.mark.parametrize("diff", ["adjoint", "ps", "fd"])
def test_layer_forward_backward_equal_materialised_jacobian(cuda, diff):
    """quantum_backward is the vector-Jacobian product of quantum_forward (ref
    test_graph.py:161-180): compared with the oracle's per-row, per-observable gradients."""
    from paper_2003_02989_b200 import graph

    rng = np.random.default_rng(91)
    model = wl.qcnn_model(8)
    data = [wl.qcnn_data_circuit(rng.uniform(-np.pi, np.pi, 8)) for _ in range(3)]
    obs = [PauliSum([PauliString(1.0, {7: "Z"})]), random_observable(rng, 8, k=3)]
    d = {"adjoint": gr.Adjoint(), "ps": gr.ParameterShift(), "fd": gr.FiniteDifference(epsilon=1e-3)}[diff]
    node = _Node(model, data, obs, d)
    pb = rng.uniform(0, 2, size=(3, len(node.symbols))).astype(np.float32).astype(np.float64)
    up = rng.normal(size=(3, 2))
    fwd = graph.quantum_forward(node, pb)
    vjp = graph.quantum_backward(node, pb, up)
    for b in range(3):
        c = node._combined(data[b])
        bind = dict(zip(node.symbols, pb[b]))
        amps = orc.simulate_amps(c, bind)
        for k, o in enumerate(obs):
            assert fwd[b, k] == pytest.approx(orc.expectation(amps, o, 8), abs=EXP)
        jac = np.stack([orc.adjoint_grad(c, o, bind)[1] for o in obs])      # [n_obs, S]
        tol = 2e-3 if diff == "fd" else GABS
        np.testing.assert_allclose(vjp[b], up[b] @ jac, atol=tol, rtol=GREL)


def test_gpu_evaluator_protocol_and_stochastic_ps(cuda):
    """The evaluator protocol (ref gradients.py:96-110) on the GPU: exact PS through a
    GpuEvaluator equals the batched PS and counts its evaluations; stochastic PS over
    coordinates / generator terms / cost terms is unbiased within 4 sigma over seeds (ref
    test_gradients.py:275-325)."""
    rng = np.random.default_rng(13)
    c = Circuit(3, [G.ry(ParamExpr("a"), 0), G.cnot_pow(ParamExpr("b", 0.7), 0, 1), G.rx(ParamExpr("a", -0.5), 2),
                    G.cz(1, 2), wl.pauli_pair_pow("X", "b", 1, 2)])
    o = PauliSum([PauliString(0.8, {0: "Z"}), PauliString(-1.2, {1: "X", 2: "Z"}), PauliString(0.5, {2: "Y"})])
    bind = {"a": 0.37, "b": -0.81}
    req = gr.GradRequest(c, o, bind)
    exact = gr.parameter_shift_grad(req)
    ev = gr.GpuEvaluator()
    viaev = gr.parameter_shift_grad(req, evaluator=ev)
    np.testing.assert_allclose(viaev.gradient, exact.gradient, atol=1e-5)
    assert ev.count == viaev.evaluations == exact.evaluations
    cfg = dict(sample_generator_terms=True, sample_cost_terms=True, sample_coordinates=True)
    draws = np.array([gr.stochastic_ps_grad(req, gr.StochasticConfig(**cfg, seed=s)).gradient for s in range(300)])
    sem = draws.std(axis=0, ddof=1) / np.sqrt(len(draws))
    assert np.all(np.abs(draws.mean(axis=0) - exact.gradient) < 4 * sem + 1e-6)
    again = gr.stochastic_ps_grad(req, gr.StochasticConfig(**cfg, seed=5)).gradient
    np.testing.assert_array_equal(again, draws[5])                         # seeded determinism


def test_layer_forward_sampled_estimator(cuda):
    """Sampled estimator in quantum_forward: per-row seeds derive_seed(seed, call_id, b, k)
    (ref graph.py:463-467) -- reproducible for the same call id, within 5 sigma of exact."""
    from paper_2003_02989_b200 import graph
    from paper_2003_02989_b200.sampling import derive_seed

    rng = np.random.default_rng(5)
    model = wl.qcnn_model(4)
    data = [wl.qcnn_data_circuit(rng.uniform(-np.pi, np.pi, 4)) for _ in range(4)]
    obs = [PauliSum([PauliString(1.0, {3: "Z"})])]
    pb = rng.uniform(0, 2, size=(4, len(circuit_symbols(model))))
    exact = graph.quantum_forward(_Node(model, data, obs, gr.Adjoint()), pb)
    n1 = _Node(model, data, obs, gr.Adjoint(), gr.Sampled(4000, seed=3))
    n2 = _Node(model, data, obs, gr.Adjoint(), gr.Sampled(4000, seed=3))
    s1, s2 = graph.quantum_forward(n1, pb), graph.quantum_forward(n2, pb)
    np.testing.assert_array_equal(s1, s2)
    assert np.all(np.abs(s1 - exact) < 5 * np.sqrt(1.0 / 4000))
    # the seeds are the reference's: row b of call 1 draws with derive_seed(3, 1, b, 0)
    c0 = n1._combined(data[0])
    syms = circuit_symbols(model)
    want = ops.sampled_expectation(c0, syms, pb[:1].astype(np.float32), obs, 4000, seed=[derive_seed(3, 1, 0, 0)])
    assert s1[0, 0] == pytest.approx(float(want[0, 0]), abs=1e-12)
