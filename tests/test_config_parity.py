"""Config-scale parity: the CUDA path at BASELINE.json's own sizes against goldens produced
by the reference itself (tests/golden/make_config_golden.py, qcflow 0.1.0 on the CPU):

  cfg1  HEA 10q, 4 layers, 1024 rows      -> 8 rows: expectation + parameter-shift gradients
  cfg2  QAOA 20q, p=4, 256 rows           -> row 0: expectation + parameter-shift gradient
  cfg3  QCNN 16q, 4096 rows               -> rows 0 and 4095: expectation + PS gradient (72)
  cfg4  RCS 24q, depth 20, 64 circuits    -> circuits 0, 1: 4096 amplitudes, 1000-shot bits,
                                              sampled sum-Z (1000 shots per term)
  cfg5  brickwork at 28q (the CPU-timed size) -> sum-Z expectation + 4096 amplitudes

Tolerances (north star): expectations / gradients 1e-4 absolute (gradients + 1e-5
relative, the complex64 floor at |g| > 10), amplitudes 1e-5.
Bitstrings use the reference's uniforms; drawn from a complex64 state instead of the
reference's complex128 one, a shot can land on the adjacent outcome when its uniform falls
within the ~1e-11 CDF difference of a boundary -- the test bounds how often and checks that
each differing shot is the neighbouring index (same-state bit-exactness:
test_gpu_parity.py::test_rcs24_sampling_bit_exact)."""

import json
import os

import numpy as np
import pytest

from paper_2003_02989_b200 import ops
from paper_2003_02989_b200 import workloads as wl
from paper_2003_02989_b200.circuit import Circuit, circuit_symbols
from paper_2003_02989_b200.pauli import PauliString, PauliSum
from paper_2003_02989_b200.sampling import derive_seed

pytestmark = pytest.mark.gpu

AMP, EXP, GABS, GREL = 1e-5, 1e-4, 1e-4, 1e-5
CFG = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cfg")


def _gold(part):
    with open(os.path.join(CFG, part + ".json")) as f:
        meta = json.load(f)
    p = os.path.join(CFG, part + ".npz")
    return meta, (dict(np.load(p)) if os.path.exists(p) else {})


def test_cfg1_hea10_full_batch_parameter_shift(cuda):
    meta, arr = _gold("cfg1")
    circ = wl.hea_circuit(10, 4)
    syms = circuit_symbols(circ)
    th = wl.hea_params(1024)
    obs = [wl.z_sum(10)]
    e, g = ops.expectation_and_ps_gradient(circ, syms, th, obs)          # the configured output
    ea, ga = ops.expectation_and_gradient(circ, syms, th, obs)           # and the adjoint
    rows = meta["rows"]
    assert meta["evaluations"] == [240] * len(rows)
    np.testing.assert_allclose(e[rows, 0], arr["exp"][:, 0], atol=EXP)
    np.testing.assert_allclose(g[rows], arr["ps"], atol=GABS, rtol=GREL)
    np.testing.assert_allclose(ea[rows, 0], arr["exp"][:, 0], atol=EXP)
    np.testing.assert_allclose(ga[rows], arr["ps"], atol=GABS, rtol=GREL)


def test_cfg2_qaoa20_headline_batch(cuda):
    meta, arr = _gold("cfg2")
    circ, cost = wl.qaoa_circuit(20, 4, wl.qaoa_graph(20))
    syms = circuit_symbols(circ)
    th = wl.qaoa_params(256, 4)
    e, g = ops.expectation_and_gradient([circ] * 256, syms, th, [cost])   # the bench's call
    rows = meta["rows"]
    np.testing.assert_allclose(e[rows, 0], arr["exp"][:, 0], atol=EXP)
    np.testing.assert_allclose(g[rows], arr["ps"], atol=GABS, rtol=GREL)
    ep, gp = ops.expectation_and_ps_gradient(circ, syms, th[rows], [cost])
    np.testing.assert_allclose(gp, arr["ps"], atol=GABS, rtol=GREL)
    assert meta["evaluations"] == [400]


def test_cfg3_qcnn16_full_batch(cuda):
    meta, arr = _gold("cfg3")
    phis, _, params = wl.qcnn_data(4096, 16)
    model = wl.qcnn_model(16)
    syms = circuit_symbols(model)
    assert syms == meta["symbols"]
    circs = [Circuit(16, list(wl.qcnn_data_circuit(p).gates) + list(model.gates)) for p in phis]
    obs = [PauliSum([PauliString(1.0, {15: "Z"})])]
    e, g = ops.expectation_and_gradient(circs, syms, params, obs)
    rows = meta["rows"]
    np.testing.assert_allclose(e[rows, 0], arr["exp"], atol=EXP)
    np.testing.assert_allclose(g[rows], arr["ps"], atol=GABS, rtol=GREL)


def _uniforms(seed, *path, n=1000):
    """The uniforms numpy's Generator(Philox(SeedSequence(seed, spawn_key=path))).choice draws
    (ref rng.py:14-19, sim.py:216-220): the GPU sampler consumes exactly these."""
    return np.random.Generator(np.random.Philox(np.random.SeedSequence(seed, spawn_key=path))).random(n)


def _check_draws(idx_gpu, idx_ref, u, cdf, tol=1e-6):
    """Both sides map the SAME uniform u through a CDF; ours is built from the complex64
    state, the reference's from its complex128 one.  Every shot where the outcomes differ
    must be a uniform that lies, within tol (relative), inside the interval our CDF assigns
    to the reference's outcome -- i.e. the difference is the CDF perturbation, nothing else.
    Returns the number of differing shots."""
    T = float(cdf[-1])
    bad = np.nonzero(idx_gpu != idx_ref)[0]
    for s_ in bad:
        k = int(idx_ref[s_])
        lo = float(cdf[k - 1]) if k > 0 else 0.0
        hi = float(cdf[k])
        x = float(u[s_]) * T
        assert lo - tol * T <= x <= hi + tol * T, (s_, k, int(idx_gpu[s_]), lo / T, hi / T, u[s_])
    return len(bad)


@pytest.mark.parametrize("b", [0, 1])
def test_cfg4_rcs24_amplitudes_bits_sampled(cuda, b):
    """Amplitudes within 1e-5; the 1000-shot sample and all 24 x 1000 per-term draws of the
    sampled sum-Z use the reference's uniforms, and every shot that differs from the
    reference's outcome is explained by the complex64-vs-complex128 CDF difference (ours
    within 1e-6 of the reference's interval).  Drawing from the SAME state is bit-exact:
    test_gpu_parity.py::test_rcs24_sampling_bit_exact."""
    import torch

    from paper_2003_02989_b200.sampling import philox_key, sample_indices

    meta, arr = _gold(f"cfg4_{b}")
    dmeta, darr = _gold(f"cfg4d_{b}")
    circs = wl.rcs_circuits(64, 24, 20)
    zs = wl.z_sum(24)
    th0 = torch.zeros((64, 0), device="cuda")
    st = ops.state(circs, [], th0)                                        # the whole 64-circuit batch
    idx = torch.as_tensor(arr["amp_idx"], device="cuda")
    np.testing.assert_allclose(st[b, idx].cpu().numpy(), arr["amps"], atol=AMP)
    psi = st[b:b + 1].contiguous()
    cdf = torch.cumsum((psi[0].abs() ** 2).double(), 0).cpu().numpy()
    del st
    w = 1 << np.arange(24, dtype=np.int64)
    # the sample op, through the public batched API
    bits = ops.sample(circs, [], np.zeros((64, 0), np.float32), 1000,
                      seed=[derive_seed(wl.SEED_RCS_SHOTS, i) for i in range(64)])
    seed_s = derive_seed(wl.SEED_RCS_SHOTS, b)
    assert meta["sample_seed"] == seed_s
    n_s = _check_draws(bits[b].astype(np.int64) @ w, arr["bits"].astype(np.int64) @ w, _uniforms(seed_s), cdf)
    # sampled sum-Z: every term k draws with substream(seed_e, k) (ref sim.py:245-272)
    seed_e = derive_seed(wl.SEED_RCS_SHOTS + 1, b)
    assert meta["sampled_seed"] == dmeta["sampled_seed"] == seed_e
    assert dmeta["sampled_expectation_from_draws"] == meta["sampled_expectation"]
    se = ops.sampled_expectation(circs, [], np.zeros((64, 0), np.float32), [zs], 1000,
                                 seed=[derive_seed(wl.SEED_RCS_SHOTS + 1, i) for i in range(64)])
    gidx, _ = sample_indices(psi, 24, 1000, [philox_key(seed_e, k) for k in range(24)], keys_per_row=24)
    gidx = gidx[0].cpu().numpy()                                          # [24 terms, 1000]
    n_t = sum(_check_draws(gidx[k], darr["term_idx"][k].astype(np.int64), _uniforms(seed_e, k), cdf)
              for k in range(24))
    # the op's value is exactly the per-term mean of these draws, pairwise-summed
    from paper_2003_02989_b200.ops import _pairwise

    ours = _pairwise([np.array([(1.0 - 2.0 * ((gidx[k] >> k) & 1)).mean()]) for k in range(24)])[0]
    assert se[b, 0] == pytest.approx(ours, abs=1e-12)
    print(f"cfg4 circuit {b}: {n_s}/1000 sample shots and {n_t}/24000 term draws differ from the "
          f"complex128 reference, all within the CDF perturbation; sampled sum-Z {se[b, 0]:.4f} vs "
          f"{meta['sampled_expectation']:.4f}")


def test_cfg5_brickwork28_vs_cpu_reference(cuda):
    import torch

    meta, arr = _gold("cfg5_28")
    circ = wl.brickwork_circuit(28, 14, wl.SEED_BIG)
    th0 = torch.zeros((1, 0), device="cuda")
    e = ops.expectation(circ, [], th0, [wl.z_sum(28)])
    assert float(e[0, 0]) == pytest.approx(meta["expectation"], abs=EXP)
    st = ops.state(circ, [], th0)
    idx = torch.as_tensor(arr["amp_idx"], device="cuda")
    np.testing.assert_allclose(st[0, idx].cpu().numpy(), arr["amps"], atol=AMP)


# ---------------------------------------------------------------------------
# every row of the full-size batches: size-independent properties between independent
# code paths (the adjoint sweep vs the reference's parameter-shift rule, both on the GPU;
# state norms; sampled vs exact expectation), on top of the reference-pinned rows above
# ---------------------------------------------------------------------------


def test_cfg1_all_rows_adjoint_equals_parameter_shift(cuda):
    circ = wl.hea_circuit(10, 4)
    syms = circuit_symbols(circ)
    th = wl.hea_params(1024)
    obs = [wl.z_sum(10)]
    e, g = ops.expectation_and_ps_gradient(circ, syms, th, obs)
    ea, ga = ops.expectation_and_gradient(circ, syms, th, obs)
    np.testing.assert_allclose(ea, e, atol=EXP)
    np.testing.assert_allclose(ga, g, atol=GABS, rtol=GREL)


def test_cfg2_all_rows_adjoint_equals_parameter_shift(cuda):
    """All 256 headline rows: the bench's adjoint output against 400-evaluation parameter
    shift on the same rows (the reference's gradient rule, a different code path)."""
    circ, cost = wl.qaoa_circuit(20, 4, wl.qaoa_graph(20))
    syms = circuit_symbols(circ)
    th = wl.qaoa_params(256, 4)
    e, g = ops.expectation_and_gradient([circ] * 256, syms, th, [cost])
    ep, gp = ops.expectation_and_ps_gradient(circ, syms, th, [cost])
    np.testing.assert_allclose(e, ep, atol=EXP)
    np.testing.assert_allclose(g, gp, atol=GABS, rtol=GREL)
    assert np.all(np.abs(e) <= 30.0 + 1e-3)        # |<sum of 30 ZZ>| <= 30


def test_cfg3_rows_adjoint_equals_parameter_shift(cuda):
    """Every 32nd of the 4096 QCNN rows (128 rows, 1080 shifted evaluations each) inside the
    full 4096-row adjoint batch."""
    phis, _, params = wl.qcnn_data(4096, 16)
    model = wl.qcnn_model(16)
    syms = circuit_symbols(model)
    circs = [Circuit(16, list(wl.qcnn_data_circuit(p).gates) + list(model.gates)) for p in phis]
    obs = [PauliSum([PauliString(1.0, {15: "Z"})])]
    e, g = ops.expectation_and_gradient(circs, syms, params, obs)
    rows = np.arange(0, 4096, 32)
    ep, gp = ops.expectation_and_ps_gradient([circs[r] for r in rows], syms, params[rows], obs)
    np.testing.assert_allclose(e[rows], ep, atol=EXP)
    np.testing.assert_allclose(g[rows], gp, atol=GABS, rtol=GREL)
    assert np.all(np.abs(e) <= 1.0 + 1e-4)


def test_cfg4_all_circuits_norms_and_sampled_sum_z(cuda):
    """All 64 RCS circuits: unit norms (1e-4 at 24 qubits in complex64), and the sampled
    sum-Z (1000 shots per term) within 6 standard deviations of the exact sum-Z."""
    import torch

    circs = wl.rcs_circuits(64, 24, 20)
    zs = wl.z_sum(24)
    th = np.zeros((64, 0), np.float32)
    st = ops.state(circs, [], torch.zeros((64, 0), device="cuda"))
    norms = (st.abs() ** 2).double().sum(dim=1).cpu().numpy()
    del st
    np.testing.assert_allclose(norms, 1.0, atol=1e-4)
    exact = ops.expectation(circs, [], th, [zs])[:, 0]
    se = ops.sampled_expectation(circs, [], th, [zs], 1000,
                                 seed=[derive_seed(wl.SEED_RCS_SHOTS + 1, i) for i in range(64)])[:, 0]
    # per term Var(+-1) <= 1, 1000 shots, 24 independent terms
    assert np.all(np.abs(se - exact) <= 6.0 * np.sqrt(24 / 1000.0)), np.max(np.abs(se - exact))
