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


@pytest.mark.parametrize("b", [0, 1])
def test_cfg4_rcs24_amplitudes_bits_sampled(cuda, b):
    import torch

    meta, arr = _gold(f"cfg4_{b}")
    circs = wl.rcs_circuits(64, 24, 20)
    zs = wl.z_sum(24)
    th0 = torch.zeros((64, 0), device="cuda")
    st = ops.state(circs, [], th0)                                        # the whole 64-circuit batch
    idx = torch.as_tensor(arr["amp_idx"], device="cuda")
    np.testing.assert_allclose(st[b, idx].cpu().numpy(), arr["amps"], atol=AMP)
    del st
    bits = ops.sample(circs, [], np.zeros((64, 0), np.float32), 1000,
                      seed=[derive_seed(wl.SEED_RCS_SHOTS, i) for i in range(64)])
    assert meta["sample_seed"] == derive_seed(wl.SEED_RCS_SHOTS, b)
    # Same uniforms, but the reference draws from its complex128 state and the GPU from the
    # complex64 one: over 2^24 outcomes their CDFs differ by ~1e-11, so a uniform landing that
    # close to a boundary picks the neighbouring index (expected ~1 shot in 1000).  Every other
    # shot is bit-identical; a differing shot is the adjacent outcome.  (Bit-exactness for the
    # SAME state is test_gpu_parity.py::test_rcs24_sampling_bit_exact.)
    w8 = 1 << np.arange(24, dtype=np.int64)
    got_idx, want_idx = bits[b].astype(np.int64) @ w8, arr["bits"].astype(np.int64) @ w8
    diff = got_idx != want_idx
    assert diff.sum() <= 5, diff.sum()
    assert np.all(np.abs(got_idx[diff] - want_idx[diff]) == 1), (got_idx[diff], want_idx[diff])
    se = ops.sampled_expectation(circs, [], np.zeros((64, 0), np.float32), [zs], 1000,
                                 seed=[derive_seed(wl.SEED_RCS_SHOTS + 1, i) for i in range(64)])
    assert meta["sampled_seed"] == derive_seed(wl.SEED_RCS_SHOTS + 1, b)
    # 24 terms x 1000 shots: the same boundary effect, each flipped shot moves one term's mean
    # by 2/1000 -- allow up to 3 such shots
    assert se[b, 0] == pytest.approx(meta["sampled_expectation"], abs=6e-3 + 1e-9)


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
