"""Seeded random circuit / observable factories for the tests (this package's gates)."""

import numpy as np

from paper_2003_02989_b200 import gates as G
from paper_2003_02989_b200 import workloads as wl
from paper_2003_02989_b200.circuit import Circuit, Gate, ParamExpr
from paper_2003_02989_b200.pauli import PauliString, PauliSum

F1 = [G.x, G.y, G.z, G.h, G.s, G.t]
P1 = [G.rx, G.ry, G.rz, G.xpow, G.ypow, G.zpow]
F2 = [G.cz, G.cnot, G.swap]


def random_unitary(d, rng):
    z = rng.normal(size=(d, d)) + 1j * rng.normal(size=(d, d))
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


def random_circuit(rng, n, depth, n_sym=0, p2=0.35):
    """Mix of fixed, concrete-parameterised, symbolic (affine, shared) and dense-matrix gates."""
    names = [f"s{i}" for i in range(n_sym)]
    gs = []
    for _ in range(depth):
        if n >= 2 and rng.random() < p2:
            a, b = (int(q) for q in rng.choice(n, 2, replace=False))
            r = rng.random()
            if r < 0.15:
                gs.append(G.cnot_pow(float(rng.uniform(-1.5, 1.5)), a, b))
            elif r < 0.3 and names:
                gs.append(G.cnot_pow(ParamExpr(names[rng.integers(n_sym)], float(rng.uniform(-1.5, 1.5)),
                                               float(rng.uniform(-.5, .5))), a, b))
            elif r < 0.45 and names:
                gs.append(wl.pauli_pair_pow("XYZ"[rng.integers(3)], names[rng.integers(n_sym)], a, b))
            elif r < 0.55:
                gs.append(Gate((a, b), matrix=random_unitary(4, rng)))
            else:
                gs.append(F2[rng.integers(3)](a, b))
        else:
            q = int(rng.integers(n))
            r = rng.random()
            if r < 0.3:
                gs.append(F1[rng.integers(6)](q))
            elif r < 0.45:
                gs.append(P1[rng.integers(6)](float(rng.uniform(-2, 2)), q))
            elif r < 0.5:
                gs.append(Gate((q,), matrix=random_unitary(2, rng)))
            elif names:
                gs.append(P1[rng.integers(6)](ParamExpr(names[rng.integers(n_sym)], float(rng.uniform(-1.5, 1.5)),
                                                        float(rng.uniform(-.5, .5))), q))
            else:
                gs.append(P1[rng.integers(6)](float(rng.uniform(-2, 2)), q))
    return Circuit(n, gs)


def random_observable(rng, n, diag=False, k=4, identity=True):
    terms = [PauliString(float(rng.uniform(-1, 1)))] if identity else []
    for _ in range(k):
        qs = rng.choice(n, size=int(rng.integers(1, min(3, n) + 1)), replace=False)
        terms.append(PauliString(float(rng.uniform(-2, 2)),
                                 {int(q): ("Z" if diag else "XYZ"[rng.integers(3)]) for q in qs}))
    return PauliSum(terms)


def rotation_circuit(rng, n, depth, n_sym):
    """Symbolic gates are single-qubit rotations only (Pauli-frame eligible adjoint); fixed
    gates of every kind (Paulis, H/S/T, CZ/CNOT/SWAP, random 1q/2q unitaries, cnot_pow)."""
    names = [f"s{i}" for i in range(n_sym)]
    gs = []
    for _ in range(depth):
        r = rng.random()
        if n >= 2 and r < 0.25:
            a, b = (int(q) for q in rng.choice(n, 2, replace=False))
            k = rng.random()
            if k < 0.2:
                gs.append(Gate((a, b), matrix=random_unitary(4, rng)))
            elif k < 0.35:
                gs.append(G.cnot_pow(float(rng.uniform(-1.5, 1.5)), a, b))
            else:
                gs.append(F2[rng.integers(3)](a, b))
        else:
            q = int(rng.integers(n))
            k = rng.random()
            if k < 0.15:
                gs.append(F1[rng.integers(6)](q))
            elif k < 0.2:
                gs.append(Gate((q,), matrix=random_unitary(2, rng)))
            elif k < 0.35:
                gs.append(P1[rng.integers(6)](float(rng.uniform(-3, 3)), q))
            else:
                gs.append(P1[rng.integers(6)](ParamExpr(names[rng.integers(n_sym)], float(rng.uniform(-1.5, 1.5)),
                                                        float(rng.uniform(-.5, .5))), q))
    return Circuit(n, gs)


def pauli_rotation_circuit(rng, n, depth, n_sym):
    """Symbolic rotations, constant Z-type rotations, Z and CZ only: every op is a normalised
    rotation or diagonal under the Pauli frame (no dense op absorbs it), so the checkpointed
    adjoint applies."""
    names = [f"s{i}" for i in range(n_sym)]
    gs = []
    for _ in range(depth):
        r = rng.random()
        if n >= 2 and r < 0.25:
            a, b = (int(q) for q in rng.choice(n, 2, replace=False))
            gs.append(G.cz(a, b))
        else:
            q = int(rng.integers(n))
            k = rng.random()
            if k < 0.05:
                gs.append(G.z(q))
            elif k < 0.2:
                gs.append((G.rz, G.zpow)[rng.integers(2)](float(rng.uniform(-3, 3)), q))
            else:
                gs.append(P1[rng.integers(6)](ParamExpr(names[rng.integers(n_sym)], float(rng.uniform(-1.5, 1.5)),
                                                        float(rng.uniform(-.5, .5))), q))
    return Circuit(n, gs)
