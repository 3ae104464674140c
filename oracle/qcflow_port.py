"""CPU ORACLE -- test infrastructure only, never the product path.

A NumPy restatement of the reference package's state-vector hot path
(``/root/reference/pkg/src/qcflow``, numpy 2.3.5 semantics), used as the
checker for the CUDA path.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.

Circuits/observables are read by duck typing (``num_qubits``, ``gates``,
``targets``, ``matrix``, ``exponent.{symbol,coeff,const}``, ``generator``,
``terms``, ``coefficient``, ``factors``), so the same objects feed this oracle,
the GPU package and (in this container) the reference itself.

Parity pinning: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by the real reference (``tests/golden/
make_golden.py``), so the oracle is pinned, not free-standing.

Every function cites the reference file:line it restates.
"""

from __future__ import annotations

import math
import os

import numpy as np

NORM_TOL = 1e-9          # sim.py:24
SHIFT = math.pi / 4.0    # gradients.py:37
_PAULI = {
    "X": np.array([[0, 1], [1, 0]], dtype=np.complex128),
    "Y": np.array([[0, -1j], [1j, 0]], dtype=np.complex128),
    "Z": np.array([[1, 0], [0, -1]], dtype=np.complex128),
}
_I2 = np.eye(2, dtype=np.complex128)
_SWAP4 = np.eye(4, dtype=np.complex128)[[0, 2, 1, 3]]


# ---------------------------------------------------------------------------
# RNG streams -- rng.py:14-27
# ---------------------------------------------------------------------------


def substream(seed: int, *path: int) -> np.random.Generator:
    """rng.py:14-19: Philox(SeedSequence(seed, spawn_key=path))."""
    if seed < 0:
        raise ValueError("seed must be non-negative")
    return np.random.Generator(np.random.Philox(np.random.SeedSequence(int(seed), spawn_key=tuple(int(p) for p in path))))


def derive_seed(seed: int, *path: int) -> int:
    """rng.py:22-27."""
    if seed < 0:
        raise ValueError("seed must be non-negative")
    return int(np.random.SeedSequence(int(seed), spawn_key=tuple(int(p) for p in path)).generate_state(1, np.uint64)[0])


# ---------------------------------------------------------------------------
# Gate matrices -- circuit.py:281-309, pauli.py:62-74
# ---------------------------------------------------------------------------


def pauli_local(factors, coefficient, targets) -> np.ndarray:
    """pauli.py:62-74: kron over ``targets`` (targets[0] = MSB)."""
    m = np.array([[coefficient]], dtype=np.complex128)
    for q in targets:
        m = np.kron(m, _PAULI.get(factors.get(q, "I"), _I2))
    return m


def gate_matrix(g, bindings=None) -> np.ndarray:
    """circuit.py:281-309: identity terms -> phase; 1 term -> cos/sin; else eigh."""
    if g.matrix is not None:
        return np.asarray(g.matrix, dtype=np.complex128)
    e = g.exponent
    if e.symbol is None:
        v = e.const
    else:
        if bindings is None or e.symbol not in bindings:
            raise KeyError(f"missing binding for symbol '{e.symbol}'")
        v = e.coeff * float(bindings[e.symbol]) + e.const
    dim = 2 ** len(g.targets)
    phase = 1.0 + 0.0j
    plain = []
    for t in g.generator.terms:
        if not t.factors:
            phase *= np.exp(-1j * v * t.coefficient)
        else:
            plain.append(t)
    if not plain:
        return phase * np.eye(dim, dtype=np.complex128)
    if len(plain) == 1:
        t = plain[0]
        eta = v * t.coefficient
        p = pauli_local(t.factors, 1.0, g.targets)
        return phase * (math.cos(eta) * np.eye(dim) - 1j * math.sin(eta) * p)
    hm = np.zeros((dim, dim), dtype=np.complex128)
    for t in plain:
        hm += pauli_local(t.factors, t.coefficient, g.targets)
    w, vec = np.linalg.eigh(hm)
    return phase * ((vec * np.exp(-1j * v * w)) @ vec.conj().T)


def resolved_ops(circuit, bindings=None):
    """sim.py:116-119 (+ resolve, circuit.py:255-265): [(matrix, targets)]."""
    return [(gate_matrix(g, bindings), tuple(g.targets)) for g in circuit.gates]


def circuit_symbols(circuit) -> list:
    """circuit.py:219-227 first-appearance order."""
    out = []
    for g in circuit.gates:
        s = None if g.exponent is None else g.exponent.symbol
        if s is not None and s not in out:
            out.append(s)
    return out


# ---------------------------------------------------------------------------
# Fusion -- fusion.py:78-176
# ---------------------------------------------------------------------------


def fuse_resolved(ops, n):
    """fusion.py:78-176: ASAP lattice, 2q anchors absorb 1q gates and a
    following same-support 2q gate; residual 1q rows fused per row."""
    for _, tg in ops:
        if len(tg) > 2:
            raise ValueError(f"fusion is defined only for gates on <= 2 qubits, got {tg}")
    front = [0] * n
    cell = {}
    steps = []
    for i, (_, tg) in enumerate(ops):
        ts = max(front[q] for q in tg)
        for q in tg:
            front[q] = ts + 1
            cell[(q, ts)] = i
        steps.append(ts)
    T = max(steps) + 1 if steps else 0
    used = [False] * len(ops)
    ctr = [0] * n
    out = []

    def emb(u, slot):
        return np.kron(u, _I2) if slot == 0 else np.kron(_I2, u)

    def canon(m, tg, a):
        return m if tg[0] == a else _SWAP4 @ m @ _SWAP4

    def fwd(row, slot, t0, m):
        t = t0
        while t < T:
            j = cell.get((row, t))
            if j is not None and not used[j]:
                mj, tj = ops[j]
                if len(tj) != 1:
                    return t, m
                m = emb(mj, slot) @ m
                used[j] = True
            t += 1
        return T, m

    for ts in range(T):
        for row in range(n):
            i = cell.get((row, ts))
            if i is None or used[i] or len(ops[i][1]) == 1:
                continue
            mat, tg = ops[i]
            a, b = sorted(tg)
            f = canon(mat, tg, a)
            used[i] = True
            for r, slot in ((a, 0), (b, 1)):
                for t in range(ts - 1, ctr[r] - 1, -1):
                    j = cell.get((r, t))
                    if j is None or used[j]:
                        continue
                    f = f @ emb(ops[j][0], slot)
                    used[j] = True
            ca, f = fwd(a, 0, ts + 1, f)
            cb, f = fwd(b, 1, ts + 1, f)
            while ca == cb and ca < T:
                j = cell.get((a, ca))
                if j is None or j != cell.get((b, cb)) or used[j]:
                    break
                f = canon(ops[j][0], ops[j][1], a) @ f
                used[j] = True
                ca, f = fwd(a, 0, ca + 1, f)
                cb, f = fwd(b, 1, cb + 1, f)
            ctr[a], ctr[b] = ca, cb
            out.append((f, (a, b)))
    for row in range(n):
        acc = None
        for t in range(T):
            j = cell.get((row, t))
            if j is None or used[j]:
                continue
            acc = ops[j][0] if acc is None else ops[j][0] @ acc
            used[j] = True
        if acc is not None:
            out.append((acc, (row,)))
    return out


# ---------------------------------------------------------------------------
# Simulation -- sim.py:27-150
# ---------------------------------------------------------------------------


def max_qubits() -> int:
    """sim.py:27-35."""
    raw = os.environ.get("QCFLOW_MAX_QUBITS")
    if raw is None:
        return 26
    try:
        return int(raw)
    except ValueError as exc:
        raise ValueError(f"bad QCFLOW_MAX_QUBITS value {raw!r}") from exc


def apply_matrix(amps, matrix, targets, n):
    """sim.py:88-105: tensordot over target axes; batch-aware."""
    k = len(targets)
    lead = amps.shape[:-1]
    nb = len(lead)
    full = amps.reshape(lead + (2,) * n)
    axes = tuple(nb + (n - 1 - q) for q in targets)
    out = np.tensordot(np.asarray(matrix).reshape((2,) * (2 * k)), full,
                       axes=(tuple(range(k, 2 * k)), axes))
    out = np.moveaxis(out, tuple(range(k)), axes)
    return np.ascontiguousarray(out).reshape(amps.shape)


def run_ops(amps, ops, n, fuse_enabled=True):
    """sim.py:122-136."""
    seq = fuse_resolved(ops, n) if fuse_enabled else ops
    for m, tg in seq:
        amps = apply_matrix(amps, m, tg, n)
    return amps


def simulate_amps(circuit, bindings=None, fuse_enabled=True, initial=None):
    """sim.py:139-150 (returns the raw c128 amplitudes; norm check sim.py:50-52)."""
    n = circuit.num_qubits
    cap = max_qubits()
    if n > cap:
        raise MemoryError(f"{n} qubits exceeds the configured cap of {cap} "
                          "(set QCFLOW_MAX_QUBITS to raise it)")
    if bindings is None and any(g.exponent is not None and g.exponent.symbol is not None
                                for g in circuit.gates):
        raise KeyError(f"circuit has unresolved symbols: {', '.join(circuit_symbols(circuit))}")
    if initial is None:
        amps = np.zeros(2 ** n, dtype=np.complex128)
        amps[0] = 1.0
    else:
        amps = np.asarray(initial, dtype=np.complex128)
    amps = run_ops(amps, resolved_ops(circuit, bindings), n, fuse_enabled)
    norm = float(np.vdot(amps, amps).real)
    if abs(norm - 1.0) > NORM_TOL:
        raise ValueError(f"state norm^2 deviates from 1 by {abs(norm - 1.0):.2e}")
    return amps


def pairwise_sum(values):
    """sim.py:162-174 deterministic pairwise tree."""
    if not values:
        return 0.0
    work = list(values)
    while len(work) > 1:
        nxt = [work[i] + work[i + 1] for i in range(0, len(work) - 1, 2)]
        if len(work) % 2:
            nxt.append(work[-1])
        work = nxt
    return work[0]


def pauli_term_values(amps, term, n):
    """sim.py:177-200: <psi|P|psi> for the coefficient-1 string; batch-aware."""
    idx = np.arange(2 ** n)
    mask = 0
    phase = np.ones(2 ** n, dtype=np.complex128)
    for q, p in term.factors.items():
        bit = (idx >> q) & 1
        if p == "Z":
            phase = phase * (1 - 2 * bit)
        elif p == "X":
            mask |= 1 << q
        else:
            mask |= 1 << q
            phase = phase * (1j * (1 - 2 * bit))
    vals = np.einsum("...i,...i->...", amps[..., idx ^ mask].conj(), phase * amps)
    resid = float(np.max(np.abs(vals.imag))) if vals.size else 0.0
    if resid > 1e-10:
        raise AssertionError(f"Pauli expectation has imaginary residue {resid:.2e}")
    return vals.real


def expectation(amps, obs, n):
    """sim.py:203-213."""
    parts = []
    for t in _terms(obs):
        if not t.factors:
            parts.append(t.coefficient)
        else:
            parts.append(t.coefficient * float(pauli_term_values(amps, t, n)))
    return float(pairwise_sum(parts))


def _terms(obs):
    if hasattr(obs, "terms"):
        return list(obs.terms)
    return [obs]


def draw_bits(amps, n, shots, rng):
    """sim.py:216-220 (Generator.choice over p = |a|^2 / sum)."""
    probs = np.abs(amps) ** 2
    probs = probs / probs.sum()
    idx = rng.choice(2 ** n, size=shots, p=probs)
    return ((idx[:, None] >> np.arange(n)[None, :]) & 1).astype(np.uint8)


def draw_indices(amps, n, shots, rng):
    """Same draw as :func:`draw_bits`, returning basis indices."""
    probs = np.abs(amps) ** 2
    probs = probs / probs.sum()
    return rng.choice(2 ** n, size=shots, p=probs)


def sample(amps, n, shots, seed):
    """sim.py:223-227."""
    if shots < 1:
        raise ValueError("shots must be >= 1")
    return draw_bits(amps, n, shots, substream(seed))


def basis_change_ops(term):
    """sim.py:230-242: H for X; Z**-0.5 then H for Y (as (matrix, targets))."""
    h = np.array([[1, 1], [1, -1]], dtype=np.complex128) / math.sqrt(2.0)
    # zpow(-0.5): exp(i*pi*t/2) * exp(-i*(pi*t/2) Z) at t=-0.5 (gates.py:109-125)
    eta = math.pi / 2.0 * -0.5
    zp = np.exp(-1j * eta * -1.0) * (math.cos(eta) * _I2 - 1j * math.sin(eta) * _PAULI["Z"])
    out = []
    for q, p in sorted(term.factors.items()):
        if p == "X":
            out.append((h, (q,)))
        elif p == "Y":
            out.append((zp, (q,)))
            out.append((h, (q,)))
    return out


def sampled_expectation(circuit, obs, shots_per_term, seed, bindings=None, fuse_enabled=True,
                        rotated_states=None):
    """sim.py:245-272.  ``rotated_states`` (optional dict term-index -> amps) lets a
    test feed externally computed basis-rotated states to the same draw path."""
    if shots_per_term < 1:
        raise ValueError("shots_per_term must be >= 1")
    n = circuit.num_qubits
    base = resolved_ops(circuit, bindings)
    parts = []
    for k, t in enumerate(_terms(obs)):
        if not t.factors:
            parts.append(t.coefficient)
            continue
        if rotated_states is not None:
            amps = rotated_states[k]
        else:
            z = np.zeros(2 ** n, dtype=np.complex128)
            z[0] = 1.0
            amps = run_ops(z, base + basis_change_ops(t), n, fuse_enabled)
        bits = draw_bits(amps, n, shots_per_term, substream(seed, k))
        eig = np.ones(shots_per_term)
        for q in t.factors:
            eig *= 1.0 - 2.0 * bits[:, q]
        parts.append(t.coefficient * float(eig.mean()))
    return float(pairwise_sum(parts))


def batch_execute(circuits, bindings_matrix, observables):
    """sim.py:275-294."""
    out = np.zeros((len(circuits), len(observables)))
    for i, c in enumerate(circuits):
        syms = circuit_symbols(c)
        row = np.atleast_1d(np.asarray(bindings_matrix[i], dtype=np.float64)) if syms else []
        if len(row) != len(syms):
            raise ValueError(f"row {i}: ragged symbol coverage ({len(row)} values for {len(syms)} symbols)")
        amps = simulate_amps(c, dict(zip(syms, row)))
        for k, o in enumerate(observables):
            out[i, k] = expectation(amps, o, c.num_qubits)
    return out


# ---------------------------------------------------------------------------
# Gradients -- gradients.py:113-326
# ---------------------------------------------------------------------------


def _strings_commute(a, b):
    """pauli.py:204-212."""
    return sum(1 for q, p in a.factors.items() if q in b.factors and b.factors[q] != p) % 2 == 0


def _occurrences(circuit, bindings, symbols):
    """gradients.py:206-221."""
    index = {s: i for i, s in enumerate(symbols)}
    occ = []
    for j, g in enumerate(circuit.gates):
        if g.exponent is None or g.exponent.symbol is None:
            continue
        ts = list(g.generator.terms)
        for a in range(len(ts)):
            for b in range(a + 1, len(ts)):
                if not _strings_commute(ts[a], ts[b]):
                    raise ValueError(
                        f"gate {j}: generator terms do not commute, so the parameter-shift "
                        "rule does not apply — use finite_difference_grad instead")
        terms = tuple(t for t in ts if t.factors and t.coefficient != 0.0)
        v = g.exponent.coeff * float(bindings[g.exponent.symbol]) + g.exponent.const
        occ.append((j, index[g.exponent.symbol], g.exponent.coeff, v, terms))
    return occ


def _term_matrix(term, eta):
    sup = tuple(sorted(term.factors))
    p = pauli_local(term.factors, 1.0, sup)
    return math.cos(eta) * np.eye(p.shape[0]) - 1j * math.sin(eta) * p, sup


def parameter_shift_grad(circuit, obs, bindings, evaluate=None):
    """gradients.py:158-165 + _ps_driver (:241-326) with all sampling off.

    Returns (gradient[S], evaluations).  ``evaluate(ops) -> float`` defaults to
    fused simulation + exact expectation (the _Evaluator Exact path, :103-110).
    """
    n = circuit.num_qubits
    symbols = circuit_symbols(circuit)
    missing = [s for s in symbols if s not in bindings]
    if missing:
        raise KeyError(f"missing binding for symbol(s): {', '.join(missing)}")
    if not symbols:
        return np.zeros(0), 0
    occs = _occurrences(circuit, bindings, symbols)
    base = resolved_ops(circuit, bindings)
    if evaluate is None:
        def evaluate(ops):
            z = np.zeros(2 ** n, dtype=np.complex128)
            z[0] = 1.0
            return expectation(run_ops(z, ops, n, True), obs, n)
    grad = np.zeros(len(symbols))
    count = 0
    for j, si, scale, v, terms in occs:
        for k, t in enumerate(terms):
            w = scale * t.coefficient
            if w == 0.0:
                continue
            f = []
            for delta in (+SHIFT, -SHIFT):
                exp_ops = [_term_matrix(tt, v * tt.coefficient + (delta if kk == k else 0.0))
                           for kk, tt in enumerate(terms)]
                f.append(evaluate(base[:j] + exp_ops + base[j + 1:]))
                count += 1
            grad[si] += w * (f[0] - f[1])
    if not np.all(np.isfinite(grad)):
        raise ValueError("gradient has non-finite entries")
    return grad, count


def finite_difference_grad(circuit, obs, bindings, scheme="central", epsilon=1e-4):
    """gradients.py:113-155."""
    n = circuit.num_qubits
    symbols = circuit_symbols(circuit)

    def f(point):
        return expectation(simulate_amps(circuit, point), obs, n)

    g = np.zeros(len(symbols))
    if scheme == "central":
        for k, s in enumerate(symbols):
            up = dict(bindings, **{s: bindings[s] + epsilon})
            dn = dict(bindings, **{s: bindings[s] - epsilon})
            g[k] = (f(up) - f(dn)) / (2 * epsilon)
    else:
        f0 = f(bindings)
        for k, s in enumerate(symbols):
            g[k] = (f(dict(bindings, **{s: bindings[s] + epsilon})) - f0) / epsilon
    return g


def pauli_sum_apply(amps, obs, n):
    """H|psi> for a Pauli sum (index/phase form of sim.py:177-200)."""
    idx = np.arange(2 ** n)
    out = np.zeros_like(amps)
    for t in _terms(obs):
        mask = 0
        phase = np.full(2 ** n, t.coefficient, dtype=np.complex128)
        for q, p in t.factors.items():
            bit = (idx >> q) & 1
            if p == "Z":
                phase = phase * (1 - 2 * bit)
            elif p == "X":
                mask |= 1 << q
            else:
                mask |= 1 << q
                phase = phase * (1j * (1 - 2 * bit))
        # (P psi)[x ^ mask] = phase(x) psi[x]
        out[..., idx ^ mask] += phase * amps
    return out


def adjoint_grad(circuit, obs, bindings):
    """Adjoint differentiation restated on the reference ops.

    The reference has no adjoint engine; this is the CPU check
    for the GPU adjoint, itself pinned against ``parameter_shift_grad``:
    dE/dtheta_s = sum_{j: sym(j)=s} coeff_j * 2 Im <lam_j| G_j |psi_j>.
    """
    n = circuit.num_qubits
    symbols = circuit_symbols(circuit)
    index = {s: i for i, s in enumerate(symbols)}
    ops = resolved_ops(circuit, bindings)
    psi = np.zeros(2 ** n, dtype=np.complex128)
    psi[0] = 1.0
    for m, tg in ops:
        psi = apply_matrix(psi, m, tg, n)
    lam = pauli_sum_apply(psi, obs, n)
    energy = float(np.vdot(psi, lam).real)
    grad = np.zeros(len(symbols))
    for j in range(len(ops) - 1, -1, -1):
        g = circuit.gates[j]
        m, tg = ops[j]
        if g.exponent is not None and g.exponent.symbol is not None:
            gm = np.zeros((2 ** len(tg),) * 2, dtype=np.complex128)
            for t in g.generator.terms:
                if t.factors:
                    gm += pauli_local(t.factors, t.coefficient, tg)
            gpsi = apply_matrix(psi, gm, tg, n)
            grad[index[g.exponent.symbol]] += g.exponent.coeff * 2.0 * float(np.vdot(lam, gpsi).imag)
        mh = m.conj().T
        psi = apply_matrix(psi, mh, tg, n)
        lam = apply_matrix(lam, mh, tg, n)
    return energy, grad
