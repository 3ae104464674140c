"""Pin the CPU oracle (oracle/qcflow_port.py) against golden vectors produced by the
real reference (tests/golden/make_golden.py).  CPU only.

Circuits are re-hydrated with this package's ``from_json`` (the host mirror of
qcflow's JSON schema, ref circuit.py:359-448), which is therefore pinned too.
"""

import json

import numpy as np
import pytest

from oracle import qcflow_port as orc
from paper_2003_02989_b200.circuit import circuit_symbols, from_json
from paper_2003_02989_b200.pauli import pauli_sum_from_obj


def _obs(s):
    return pauli_sum_from_obj(json.loads(s))


def test_known_answers(golden):
    meta, arr = golden
    bell = from_json(meta["cases"]["bell"]["circuit"])
    amps = orc.simulate_amps(bell)
    np.testing.assert_allclose(amps, arr["bell/amps"], atol=1e-12)
    np.testing.assert_allclose(amps, [2 ** -0.5, 0, 0, 2 ** -0.5], atol=1e-12)
    c = from_json(meta["cases"]["xpow_ladder"]["circuit"])
    out = orc.batch_execute([c] * 3, meta["cases"]["xpow_ladder"]["rows"], [_obs('[{"coeff": 1.0, "paulis": {"0": "Z"}}]')])
    np.testing.assert_allclose(out, arr["xpow_ladder/out"], atol=1e-12)
    np.testing.assert_allclose(out, [[1], [-1], [1]], atol=1e-12)


@pytest.mark.parametrize("i", range(8))
def test_concrete_states_fusion_expectations(golden, i):
    meta, arr = golden
    case = meta["cases"][f"concrete{i}"]
    c = from_json(case["circuit"])
    n = c.num_qubits
    amps = orc.simulate_amps(c)
    np.testing.assert_allclose(amps, arr[f"concrete{i}/amps"], atol=1e-12)
    np.testing.assert_allclose(orc.simulate_amps(c, fuse_enabled=False), arr[f"concrete{i}/amps_unfused"], atol=1e-12)
    fz = orc.fuse_resolved(orc.resolved_ops(c), n)
    assert [list(t) for _, t in fz] == case["fused_targets"]
    for (m, _), want in zip(fz, arr[f"concrete{i}/fused_mats"]):
        np.testing.assert_allclose(m, want[: m.shape[0], : m.shape[0]], atol=1e-12)
    for o, e in zip(case["observables"], case["expectations"]):
        assert orc.expectation(amps, _obs(o), n) == pytest.approx(e, abs=1e-12)


@pytest.mark.parametrize("i", range(8))
def test_sampler_and_sampled_expectation_bit_exact(golden, i):
    meta, arr = golden
    case = meta["cases"][f"concrete{i}"]
    c = from_json(case["circuit"])
    n = c.num_qubits
    amps = orc.simulate_amps(c)
    bits = orc.sample(amps, n, case["shots"], case["sample_seed"])
    np.testing.assert_array_equal(bits, arr[f"concrete{i}/bits"])
    obs = _obs(case["observables"][0])
    assert orc.sampled_expectation(c, obs, case["shots_per_term"], case["sampled_seed"]) == case["sampled_expectation"]


@pytest.mark.parametrize("i", range(4))
def test_parameter_shift_and_fd(golden, i):
    meta, arr = golden
    case = meta["cases"][f"symbolic{i}"]
    c = from_json(case["circuit"])
    obs = _obs(case["observable"])
    assert circuit_symbols(c) == case["symbols"]
    b = dict(zip(case["symbols"], case["bindings"]))
    g, n_eval = orc.parameter_shift_grad(c, obs, b)
    np.testing.assert_allclose(g, arr[f"symbolic{i}/ps"], atol=1e-12)
    assert n_eval == case["ps_evaluations"]
    np.testing.assert_allclose(orc.finite_difference_grad(c, obs, b), arr[f"symbolic{i}/fd"], atol=1e-9)
    # the adjoint restatement equals the reference's PS gradient
    e, ga = orc.adjoint_grad(c, obs, b)
    np.testing.assert_allclose(ga, arr[f"symbolic{i}/ps"], atol=1e-10)
    assert e == pytest.approx(case["expectation"], abs=1e-12)


def test_config_families(golden):
    meta, arr = golden
    cfg = meta["configs"]
    for name in ("hea", "qaoa"):
        c = from_json(cfg[name]["circuit"])
        o = _obs(cfg[name]["observable"])
        rows = np.array(cfg[name]["rows"])
        np.testing.assert_allclose(orc.batch_execute([c, c], rows, [o]), arr[f"{name}/exp"], atol=1e-12)
        for r, want in zip(rows, arr[f"{name}/ps"]):
            b = dict(zip(circuit_symbols(c), r))
            np.testing.assert_allclose(orc.adjoint_grad(c, o, b)[1], want, atol=1e-10)
    c = from_json(cfg["qcnn"]["circuit"])
    o = _obs(cfg["qcnn"]["observable"])
    b = dict(zip(circuit_symbols(c), cfg["qcnn"]["row"]))
    np.testing.assert_allclose(orc.adjoint_grad(c, o, b)[1], arr["qcnn/ps"], atol=1e-10)
    c = from_json(cfg["rcs"]["circuit"])
    amps = orc.simulate_amps(c)
    np.testing.assert_allclose(amps, arr["rcs/amps"], atol=1e-12)
    np.testing.assert_array_equal(orc.sample(amps, c.num_qubits, 200, cfg["rcs"]["seed"]), arr["rcs/bits"])
    assert orc.sampled_expectation(c, _obs(cfg["rcs"]["observable"]), 300, cfg["rcs"]["seed"]) == cfg["rcs"]["sampled"]
    c = from_json(cfg["big"]["circuit"])
    assert orc.expectation(orc.simulate_amps(c), _obs(cfg["big"]["observable"]), 12) == pytest.approx(
        cfg["big"]["expectation"], abs=1e-12)


def _philox_uniforms(key, count):
    """Host restatement of the device stream (csrc/qf_capi.cu philox_uniform)."""
    M0, M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
    W0, W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
    mask = (1 << 64) - 1
    out = []
    for s in range(count):
        c = [s // 4 + 1, 0, 0, 0]
        k0, k1 = key
        for r in range(10):
            if r:
                k0, k1 = (k0 + W0) & mask, (k1 + W1) & mask
            p0, p1 = M0 * c[0], M1 * c[2]
            c = [(p1 >> 64) ^ c[1] ^ k0, p1 & mask, (p0 >> 64) ^ c[3] ^ k1, p0 & mask]
        out.append((c[s % 4] >> 11) * 2.0 ** -53)
    return out


def test_philox_stream_matches_numpy(golden):
    from paper_2003_02989_b200.sampling import philox_key

    for rec in golden[0]["philox"]:
        key = philox_key(rec["seed"], *rec["path"])
        assert list(key) == rec["key"]
        assert _philox_uniforms(key, len(rec["uniforms"])) == rec["uniforms"]
