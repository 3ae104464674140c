"""Host-side logic on the CPU: IR mirror, recipes, and the planner's device programs
executed by a NumPy emulator of the kernels' descriptor semantics vs the oracle."""

import json

import numpy as np
import pytest

import plan_emulator as em
from circuits import random_circuit, random_observable
from oracle import qcflow_port as orc
from paper_2003_02989_b200 import gates as G
from paper_2003_02989_b200 import planner as pl
from paper_2003_02989_b200 import workloads as wl
from paper_2003_02989_b200.circuit import Circuit, ParamExpr, circuit_symbols, from_json, gate_matrix, resolve, to_json
from paper_2003_02989_b200.pauli import PauliString, PauliSum, pauli_sum_to_obj


def test_gate_library_matches_oracle_gate_matrix():
    rng = np.random.default_rng(0)
    for fn in (G.rx, G.ry, G.rz, G.xpow, G.ypow, G.zpow):
        g = fn(float(rng.uniform(-3, 3)), 0)
        np.testing.assert_allclose(gate_matrix(g), orc.gate_matrix(g), atol=1e-13)
    g = G.cnot_pow(0.37, 1, 0)
    np.testing.assert_allclose(gate_matrix(g), orc.gate_matrix(g), atol=1e-13)
    np.testing.assert_allclose(gate_matrix(G.cnot_pow(1.0, 0, 1)), G.FIXED_MATRICES["cnot"], atol=1e-13)
    np.testing.assert_allclose(gate_matrix(G.xpow(1.0, 0)), G.FIXED_MATRICES["x"], atol=1e-13)


def test_json_round_trip_and_errors():
    rng = np.random.default_rng(1)
    c = random_circuit(rng, 5, 30, n_sym=3)
    c2 = from_json(to_json(c))
    assert c2.num_qubits == c.num_qubits and len(c2) == len(c)
    assert circuit_symbols(c2) == circuit_symbols(c)
    with pytest.raises(ValueError, match="gates\\[0\\]"):
        from_json('{"num_qubits": 2, "gates": [{"targets": [0]}]}')
    with pytest.raises(ValueError, match="invalid JSON"):
        from_json("{")
    with pytest.raises(KeyError):
        resolve(c, {})


def test_workload_recipes_match_reference_built_circuits(golden):
    meta, _ = golden
    cfg = meta["configs"]
    assert json.loads(to_json(wl.hea_circuit(6, 2))) == json.loads(cfg["hea"]["circuit"])
    qa, cost = wl.qaoa_circuit(10, 2, [tuple(e) for e in cfg["qaoa"]["edges"]])
    assert json.loads(to_json(qa)) == json.loads(cfg["qaoa"]["circuit"])
    assert pauli_sum_to_obj(cost) == json.loads(cfg["qaoa"]["observable"])
    assert json.loads(to_json(wl.brickwork_circuit(10, 6, seed=401))) == json.loads(cfg["rcs"]["circuit"])


def _check_program(circ, obs, n, theta, adjoint_obs_diag=True, block=False):
    syms = circuit_symbols(circ)
    si = {s: i for i, s in enumerate(syms)}
    infos = pl.analyse(circ, si)
    diag = all(all(p == "Z" for p in t.factors.values()) for t in obs.terms)
    nonid = PauliSum([t for t in obs.terms if t.factors])
    prog = pl.build_program(circ, infos, n, adjoint=False, observables=[nonid], obs_diag_ids=[0] if diag else [])
    em.check_invariants(prog)
    fixed, consts = pl.concrete_tables([circ], infos)
    mats, angs = em.build_tables(prog, theta, fixed, consts)
    coefs = np.array([t.coefficient for t in nonid.terms])
    psi, slots = em.run_forward(prog, mats, angs, theta.shape[0], n, coefs)
    ident = sum(t.coefficient for t in obs.terms if not t.factors)
    for b in range(theta.shape[0]):
        bind = dict(zip(syms, theta[b]))
        ref = orc.simulate_amps(circ, bind)
        np.testing.assert_allclose(psi[b, : 1 << circ.num_qubits], ref, atol=1e-12)
        if diag:
            E = em.slots_to_cols(slots, prog.obs_slots, 1)[b, 0] + ident
            assert E == pytest.approx(orc.expectation(ref, obs, circ.num_qubits), abs=1e-10)
    if not syms or not diag:
        return prog
    infos_a = pl.analyse(circ, si)
    adj = pl.build_program(circ, infos_a, n, adjoint=True, observables=[nonid], lam_diag=True, block=block)
    em.check_invariants(adj)
    fixed, consts = pl.concrete_tables([circ], infos_a)
    mats_a, angs_a = em.build_tables(adj, theta, fixed, consts)
    sl = em.run_adjoint(adj, mats_a, angs_a, theta.shape[0], n, psi, None, np.tile(coefs, (theta.shape[0], 1)))
    grads = em.slots_to_cols(sl, adj.grad_slots, len(syms))
    if block:
        assert len(adj.blocks) > 0
        grads = grads + em.block_grads(adj, mats_a, sl, len(syms))
    for b in range(theta.shape[0]):
        _, g = orc.adjoint_grad(circ, obs, dict(zip(syms, theta[b])))
        np.testing.assert_allclose(grads[b], g, atol=1e-5)  # float32 generator weights in the program
    return prog


@pytest.mark.parametrize("seed,n", [(0, 10), (1, 11), (2, 13), (3, 14), (4, 15), (5, 6)])
def test_planner_programs_emulated_vs_oracle(seed, n):
    rng = np.random.default_rng(seed)
    circ = random_circuit(rng, n, 90, n_sym=4)
    n_eff = max(n, pl.N_MIN)
    theta = rng.uniform(-3, 3, size=(2, len(circuit_symbols(circ))))
    _check_program(circ, random_observable(rng, n, diag=True), n_eff, theta)


def test_planner_qaoa_pass_structure():
    circ, cost = wl.qaoa_circuit(20, 4, wl.qaoa_graph(20))
    si = {s: i for i, s in enumerate(circuit_symbols(circ))}
    prog = pl.build_program(circ, pl.analyse(circ, si), 20, adjoint=False, observables=[cost], obs_diag_ids=[0])
    adj = pl.build_program(circ, pl.analyse(circ, si), 20, adjoint=True, observables=[cost], lam_diag=True)
    # p+1 passes is the minimum for 20 qubits with 13-qubit tiles (SURVEY 8(d) pass-count targets)
    assert prog.stats["passes"] == 5 and prog.stats["product_init"] == 20
    assert adj.stats["passes"] == 5


def test_planner_qaoa_small_emulated():
    circ, cost = wl.qaoa_circuit(14, 2, wl.qaoa_graph(14, seed=2))
    _check_program(circ, cost, 14, wl.qaoa_params(2, 2).astype(np.float64))


def test_planner_qcnn_and_brickwork_emulated():
    model = wl.qcnn_model(8)
    data = wl.qcnn_data_circuit(np.linspace(-3, 3, 8))
    full = Circuit(8, tuple(data.gates) + tuple(model.gates))
    rng = np.random.default_rng(9)
    theta = rng.uniform(0, 2, size=(1, len(circuit_symbols(full))))
    _check_program(full, PauliSum([PauliString(1.0, {7: "Z"})]), 10, theta)
    bw = wl.brickwork_circuit(12, 5, seed=3)
    _check_program(bw, wl.z_sum(12), 12, np.zeros((1, 0)))


@pytest.mark.parametrize("adjoint", [False, True])
def test_frame_programs_event_invariants(adjoint):
    """Pauli-frame programs (planner.build_program(frame=True)): one frame event per dense /
    diagonal / observable op, in execution order, with matching classes and x-mask columns."""
    from circuits import random_circuit
    from paper_2003_02989_b200.engine import _Term, _TermList

    rng = np.random.default_rng(17 + adjoint)
    c = random_circuit(rng, 11, 160, n_sym=4)
    syms = circuit_symbols(c)
    si = {s: i for i, s in enumerate(syms)}
    obs = _TermList([_Term({0: "Z", 3: "Z"}, 1.0), _Term({5: "Z"}, 0.5)])
    if adjoint:
        prog = pl.build_program(c, pl.analyse(c, si), 11, adjoint=True, observables=[obs], lam_diag=True, frame=True)
    else:
        prog = pl.build_program(c, pl.analyse(c, si), 11, adjoint=False, observables=[obs], obs_diag_ids=[0],
                                frame=True)
    assert prog.frame
    ev = np.array([e for e in prog.frame_events if int(e[0]) != pl.EV_PASS])
    assert sum(int(e[0]) == pl.EV_PASS for e in prog.frame_events) == len(prog.passes)
    kinds = {pl.OP_DENSE1: {pl.EV_NX, pl.EV_NY, pl.EV_ABS1}, pl.OP_DENSE2: {pl.EV_ABS2, pl.EV_NP},
             pl.OP_DIAG: {pl.EV_DIAG}, pl.OP_OBS: {pl.EV_OBS}}
    assert len(ev) == len(prog.ops)
    for op, e in zip(prog.ops, ev):
        k, cls = int(op[0]), int(op[9])
        assert int(e[0]) in kinds[k]
        if k in (pl.OP_DENSE1, pl.OP_DENSE2):
            assert int(e[3]) == int(op[3])                   # the op's matrix slab
            assert int(e[4]) == int(op[7])                   # its gradient slot
            assert (int(e[0]) in (pl.EV_NX, pl.EV_NY, pl.EV_NP)) == (cls in (pl.CLS_NX, pl.CLS_NY, pl.CLS_NP))
            assert cls != pl.CLS_XLIKE                        # absorbed X frames would break it
        else:
            assert int(op[11]) >= 0 and int(e[5]) == int(op[11])
            assert prog.recipe["term_src"].reshape(-1, 2)[int(op[11])][0] == 2
    if adjoint:
        assert any(int(e[0]) == pl.EV_NP for e in ev)        # pauli_pair_pow X/Y couplings


@pytest.mark.parametrize("n", [4, 8])
def test_block_fused_adjoint_emulated_vs_oracle(n):
    """Block-fused adjoint programs (planner.build_ops(block=True)) on the emulator: the
    two-point matrices A and the per-factor traces of qf_block_grads give the oracle's
    gradients (QCNN: conv blocks of 15 symbolic gates incl. a ZZ pair, ring-closed bricks)."""
    phis, _, params = wl.qcnn_data(2, n)
    model = wl.qcnn_model(n)
    circ = Circuit(n, list(wl.qcnn_data_circuit(phis[0]).gates) + list(model.gates))
    theta = params[:1, :len(circuit_symbols(circ))].astype(np.float64)
    obs = PauliSum([PauliString(1.0, {n - 1: "Z"}), PauliString(0.3, {0: "Z", 1: "Z"})])
    _check_program(circ, obs, max(n, pl.N_MIN), theta, block=True)


def test_block_mode_keeps_per_gate_programs_where_blocks_do_not_pay():
    """build_ops(block=True): QAOA (single-symbol rotations, ZZ phase layers) is op-for-op the
    per-gate adjoint program; a QCNN conv block becomes one two-qubit block of >= 3 symbolic
    factors; one-qubit runs are split back to one op per gate."""
    circ, cost = wl.qaoa_circuit(12, 3, wl.qaoa_graph(12))
    si = {s: i for i, s in enumerate(circuit_symbols(circ))}
    a = pl.build_ops(pl.analyse(circ, si), True, block=False)
    b = pl.build_ops(pl.analyse(circ, si), True, block=True)
    assert [(o.kind, o.qubits, o.factors, o.gates) for o in a] == [(o.kind, o.qubits, o.factors, o.gates) for o in b]
    model = wl.qcnn_model(4)
    si = {s: i for i, s in enumerate(circuit_symbols(model))}
    infos = pl.analyse(model, si)
    ops_b = pl.build_ops(infos, True, block=True)
    blocks = [o for o in ops_b if o.symbolic and len(o.factors) > 1]
    assert blocks and all(o.kind == pl.OP_DENSE2 for o in blocks)
    assert all(sum(infos[g].symbolic for g in o.factors) >= pl.BLOCK_MIN_SYMBOLIC for o in blocks)
    assert all(len(o.factors) == 1 for o in ops_b if o.kind == pl.OP_DENSE1)
    # every gate appears exactly once
    seen = sorted(g for o in ops_b for g in (o.factors or o.gates))
    assert seen == list(range(len(infos)))


def test_uniform_batch_is_a_list_of_one_circuit():
    from paper_2003_02989_b200.engine import UniformBatch

    c = wl.hea_circuit(4, 1)
    u = UniformBatch(c, 5)
    assert len(u) == 5 and all(x is c for x in u) and u.circuit is c and isinstance(u, list)


@pytest.mark.parametrize("seed,n", [(0, 6), (1, 8), (2, 10), (3, 11)])
def test_block_fused_adjoint_random_circuits_emulated(seed, n):
    """Block-fused adjoint on random circuits (symbolic cnot_pow / Pauli-pair gates, fixed
    dense gates and rotations mixed into two-qubit blocks), emulated against the oracle."""
    rng = np.random.default_rng(500 + seed)
    circ = random_circuit(rng, n, 120, n_sym=5, p2=0.5)
    theta = rng.uniform(-2, 2, size=(2, len(circuit_symbols(circ))))
    syms = circuit_symbols(circ)
    si = {s: i for i, s in enumerate(syms)}
    if not any(o.symbolic and len(o.factors) > 1 for o in pl.build_ops(pl.analyse(circ, si), True, block=True)):
        pytest.skip("no block formed")
    _check_program(circ, random_observable(rng, n, diag=True), max(n, pl.N_MIN), theta, block=True)


@pytest.mark.parametrize("n,depth,seed", [(16, 8, 3), (20, 6, 5)])
def test_relabelled_passes_emulated_vs_oracle(n, depth, seed, monkeypatch):
    """planner.plan_passes_remap (plan-specialised forward programs): each pass stores its tile
    permuted so the next pass's qubits sit on the lane bits; fewer passes than the fixed
    layout, the same state (logical layout via Program.final_pos) and the same sum-Z value."""
    circ = wl.brickwork_circuit(n, depth, seed)
    infos = pl.analyse(circ, {})
    zs = wl.z_sum(n)
    monkeypatch.setattr(pl, "REMAP", True)
    plain = pl.build_program(circ, pl.analyse(circ, {}), n, adjoint=False, observables=[zs], obs_diag_ids=[0])
    prog = pl.build_program(circ, infos, n, adjoint=False, observables=[zs], obs_diag_ids=[0], jit=True)
    assert prog.stats["remapped"] and prog.final_pos is not None
    assert len(prog.passes) < len(plain.passes), (len(prog.passes), len(plain.passes))
    em.check_invariants(prog)
    fixed, consts = pl.concrete_tables([circ], infos)
    mats, angs = em.build_tables(prog, np.zeros((1, 0)), fixed, consts)
    psi, slots = em.run_forward(prog, mats, angs, 1, n, np.ones(n))
    ref = orc.simulate_amps(circ, {})
    np.testing.assert_allclose(em.logical_state(psi, prog, n)[0], ref, atol=1e-12)
    E = em.slots_to_cols(slots, prog.obs_slots, 1)[0, 0]
    assert E == pytest.approx(orc.expectation(ref, zs, n), abs=1e-10)


def test_lane_ops_merge_last_stage(monkeypatch):
    """Lane ops (warp-shuffle X rotations on the edge layout's lane bits): the QAOA headline's
    forward and backward passes lose one register stage each, the ops of every pass are the
    same, and lane ops sit on thread bits 0..3 of a pass's last planner stage only."""
    circ, cost = wl.qaoa_circuit(20, 4, wl.qaoa_graph(20))
    si = {s: i for i, s in enumerate(circuit_symbols(circ))}

    def build(adjoint, lanes):
        monkeypatch.setattr(pl, "LANE_OPS", lanes)
        kw = dict(lam_diag=True) if adjoint else dict(obs_diag_ids=[0])
        return pl.build_program(circ, pl.analyse(circ, si), 20, adjoint=adjoint, observables=[cost], frame=True,
                                jit=True, **kw)

    def pass_ops(prog):
        out = []
        for p in prog.passes:
            qs = []
            for s_ in range(p[0], p[1]):
                st = prog.stages[s_]
                for o in prog.ops[st[48]:st[49]]:
                    if o[0] == pl.OP_DENSE1:
                        qs.append(int(st[8 + o[15] - 1]) if o[15] else int(st[o[1]]))
            out.append(sorted(qs))
        return out

    for adjoint in (False, True):
        plain, lane = build(adjoint, 0), build(adjoint, 8)
        em.check_invariants(lane)
        assert plain.stats["lane_ops"] == 0 and lane.stats["lane_ops"] > 0
        assert sum(lane.stats["stages_per_pass"]) < sum(plain.stats["stages_per_pass"])
        assert pass_ops(lane) == pass_ops(plain)
        for p in lane.passes:
            edge = p[1] - 1 if not adjoint else p[0]      # the planner's last stage
            for s_ in range(p[0], p[1]):
                st = lane.stages[s_]
                for o in lane.ops[st[48]:st[49]]:
                    if o[15]:
                        assert s_ == edge and 1 <= o[15] <= 4 and o[9] == pl.CLS_NX
