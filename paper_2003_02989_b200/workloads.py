"""Seeded synthetic workloads for BASELINE.json's five configurations.

Every recipe takes a ``lib`` namespace (``Circuit, Gate, ParamExpr, PauliString,
PauliSum, exponential_circuit`` plus the gate constructors) so the *same code*
builds the circuit with this package (default) or with the reference package
(``tests/golden/make_golden.py`` passes ``qcflow``), which is how the oracle,
the reference and the GPU path are guaranteed to consume identical circuits.

Parameters are drawn as float32 from ``np.random.default_rng(seed)`` and are
handed to the CPU side as float64 casts of those float32 values.
"""

from __future__ import annotations

import math
import types

import numpy as np

SEED_HEA = 1
SEED_QAOA_GRAPH = 2
SEED_QAOA_PARAMS = 20
SEED_QCNN = 3
SEED_RCS = 4
SEED_RCS_SHOTS = 40
SEED_BIG = 5


def default_lib():
    from . import circuit, gates, pauli

    ns = types.SimpleNamespace()
    for mod in (circuit, pauli, gates):
        for k in dir(mod):
            if not k.startswith("_"):
                setattr(ns, k, getattr(mod, k))
    return ns


def _lib(lib):
    return default_lib() if lib is None else lib


# --- cfg1: hardware-efficient ansatz ---------------------------------------


def hea_circuit(n=10, layers=4, lib=None):
    """Per layer: rx, ry, rz (distinct symbols) on each qubit, then a CZ ladder."""
    L = _lib(lib)
    gs = []
    for l in range(layers):
        for q in range(n):
            for ax, fn in (("x", L.rx), ("y", L.ry), ("z", L.rz)):
                gs.append(fn(f"t{l}_{q}_{ax}", q))
        gs += [L.cz(q, q + 1) for q in range(n - 1)]
    return L.Circuit(n, gs)


def z_sum(n, lib=None):
    L = _lib(lib)
    return L.PauliSum([L.PauliString(1.0, {q: "Z"}) for q in range(n)])


def hea_params(batch=1024, n=10, layers=4, seed=SEED_HEA):
    rng = np.random.default_rng(seed)
    return rng.uniform(0.0, 2.0 * np.pi, size=(batch, layers * n * 3)).astype(np.float32)


# --- cfg2: QAOA MaxCut -----------------------------------------------------


def qaoa_graph(n=20, seed=SEED_QAOA_GRAPH):
    import networkx as nx

    g = nx.random_regular_graph(3, n, seed=seed)
    return sorted(tuple(sorted((int(u), int(v)))) for u, v in g.edges())


def qaoa_circuit(n=20, p=4, edges=None, lib=None):
    """H^n, then p x [exp(-i g sum_E ZZ), exp(-i b sum_q X)] via exponential_circuit."""
    L = _lib(lib)
    if edges is None:
        edges = qaoa_graph(n)
    cost = L.PauliSum([L.PauliString(1.0, {u: "Z", v: "Z"}) for u, v in edges])
    mixer = L.PauliSum([L.PauliString(1.0, {q: "X"}) for q in range(n)])
    gs = [L.h(q) for q in range(n)]
    for l in range(p):
        gs += list(L.exponential_circuit([cost], [f"gamma_{l}"], num_qubits=n).gates)
        gs += list(L.exponential_circuit([mixer], [f"beta_{l}"], num_qubits=n).gates)
    return L.Circuit(n, gs), cost


def qaoa_params(batch=256, p=4, seed=SEED_QAOA_PARAMS):
    rng = np.random.default_rng(seed)
    return rng.uniform(0.0, np.pi, size=(batch, 2 * p)).astype(np.float32)


# --- cfg3: QCNN -------------------------------------------------------------


def pauli_pair_pow(letter, exponent, q0, q1, lib=None):
    L = _lib(lib)
    gen = L.PauliSum([L.PauliString(1.0, {q0: letter, q1: letter}), L.PauliString(-1.0)])
    return L.Gate((q0, q1), exponent=L.ParamExpr(exponent).scaled(math.pi / 2.0), generator=gen)


def _two_qubit_block(q0, q1, syms, L):
    gs = [L.xpow(syms[0], q0), L.ypow(syms[1], q0), L.zpow(syms[2], q0)]
    gs += [L.xpow(syms[3], q1), L.ypow(syms[4], q1), L.zpow(syms[5], q1)]
    gs += [pauli_pair_pow(ch, syms[6 + k], q0, q1, L) for k, ch in enumerate("ZYX")]
    gs += [L.xpow(syms[9], q0), L.ypow(syms[10], q0), L.zpow(syms[11], q0)]
    gs += [L.xpow(syms[12], q1), L.ypow(syms[13], q1), L.zpow(syms[14], q1)]
    return gs


def _controlled_rot(letter, sym, c, t, L):
    gen = L.PauliSum([L.PauliString(0.25, {t: letter}), L.PauliString(-0.25, {c: "Z", t: letter})])
    return L.Gate((c, t), exponent=L.ParamExpr(sym), generator=gen)


def qcnn_model(n=16, lib=None):
    """conv (15 shared symbols, both brick offsets, ring-closed) + pool (CRz CRy CRz)."""
    L = _lib(lib)
    gs = []
    active = list(range(n))
    level = 0
    while len(active) > 1:
        cs = [f"c{level}_{k}" for k in range(15)]
        ps = [f"p{level}_{k}" for k in range(3)]
        for a, b in zip(active[0::2], active[1::2]):
            gs += _two_qubit_block(a, b, cs, L)
        for a, b in zip(active[1::2], active[2::2] + [active[0]]):
            gs += _two_qubit_block(a, b, cs, L)
        half = len(active) // 2
        for src, snk in zip(active[:half], active[half:]):
            gs += [_controlled_rot("Z", ps[0], src, snk, L), _controlled_rot("Y", ps[1], src, snk, L),
                   _controlled_rot("Z", ps[2], src, snk, L)]
        active = active[half:]
        level += 1
    return L.Circuit(n, gs)


def qcnn_data_circuit(phis, lib=None):
    """Cluster state (H all, CZ ring) then rx(phi_i) on qubit i."""
    L = _lib(lib)
    n = len(phis)
    gs = [L.h(q) for q in range(n)] + [L.cz(q, (q + 1) % n) for q in range(n)]
    gs += [L.rx(float(phis[q]), q) for q in range(n)]
    return L.Circuit(n, gs)


def qcnn_data(batch=4096, n=16, seed=SEED_QCNN):
    rng = np.random.default_rng(seed)
    phis = rng.uniform(-np.pi, np.pi, size=(batch, n)).astype(np.float32)
    labels = np.where((np.abs(phis) < np.pi / 2).sum(axis=1) * 2 > n, 1.0, -1.0)
    params = rng.uniform(0.0, 2.0, size=(batch, 72)).astype(np.float32)
    return phis, labels, params


# --- cfg4 / cfg5: random brickwork -----------------------------------------


def sqrt_w_matrix():
    w = np.array([[0, np.exp(-0.25j * np.pi)], [np.exp(0.25j * np.pi), 0]])
    return np.exp(0.25j * np.pi) / math.sqrt(2.0) * (np.eye(2) - 1j * w)


def fsim_matrix(theta, phi):
    c, s = math.cos(theta), math.sin(theta)
    return np.array([[1, 0, 0, 0], [0, c, -1j * s, 0], [0, -1j * s, c, 0],
                     [0, 0, 0, np.exp(-1j * phi)]], dtype=np.complex128)


def brickwork_circuit(n, depth, seed, lib=None):
    """Per layer: one of {sqrt X, sqrt Y, sqrt W} per qubit, then fSim on (q, q+1), q = layer mod 2."""
    L = _lib(lib)
    rng = np.random.default_rng(seed)
    sw = sqrt_w_matrix()
    gs = []
    for layer in range(depth):
        for q in range(n):
            k = int(rng.integers(3))
            if k == 0:
                gs.append(L.xpow(0.5, q))
            elif k == 1:
                gs.append(L.ypow(0.5, q))
            else:
                gs.append(L.Gate((q,), name="sqrt_w", matrix=sw))
        for q in range(layer % 2, n - 1, 2):
            th, ph = rng.uniform(0.0, 2.0 * np.pi, size=2)
            gs.append(L.Gate((q, q + 1), name="fsim", matrix=fsim_matrix(th, ph)))
    return L.Circuit(n, gs)


def rcs_circuits(batch=64, n=24, depth=20, seed=SEED_RCS, lib=None):
    return [brickwork_circuit(n, depth, seed * 100_003 + b, lib) for b in range(batch)]
