"""Differentiators on the GPU engine, behind the reference's gradient API (qcflow/gradients.py).

* ``adjoint_grad`` / ``Adjoint`` -- new: one forward + one backward sweep
  (tile-pass ADJ kernels).  The reference lists adjoint differentiation as a
  non-goal; its oracle is the exact parameter-shift gradient.
* ``parameter_shift_grad`` / ``ParameterShift`` -- the reference's exact PS rule
  (gradients.py:158-165, driver :241-326): every symbolic gate is rewritten as a
  product of per-term exponentials and each term angle is shifted by +-pi/4.  Here all
  ``2*sum_occ K`` shifted circuits share one topology (each term angle is its own
  pseudo-parameter column), so the whole PS gradient is ONE batched execution.
* ``finite_difference_grad`` -- gradients.py:113-155, shifted points as batch rows.
* ``stochastic_ps_grad`` -- gradients.py:168-174 with the reference's sampling axes,
  evaluated through :class:`GpuEvaluator` (the evaluator protocol, :96-110).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Mapping

import numpy as np
import torch

from .circuit import Circuit, Gate, ParamExpr, circuit_symbols, normalize_bindings
from .pauli import PauliString, PauliSum, all_terms_commute, as_pauli_sum
from .sampling import derive_seed

CENTRAL = "central"
FORWARD = "forward"
SHIFT = math.pi / 4.0


@dataclass(frozen=True)
class Exact:
    """Exact expectation values."""


@dataclass(frozen=True)
class Sampled:
    shots: int
    seed: int = 0

    def __post_init__(self):
        if self.shots < 1:
            raise ValueError("shots must be >= 1")
        if self.seed < 0:
            raise ValueError("seed must be non-negative")


@dataclass(frozen=True)
class GradRequest:
    circuit: Circuit
    observable: object
    bindings: Mapping
    estimator: object = Exact()


@dataclass
class GradResult:
    gradient: np.ndarray
    evaluations: int
    degenerate_sampling: bool = False


@dataclass(frozen=True)
class StochasticConfig:
    sample_generator_terms: bool = False
    sample_cost_terms: bool = False
    sample_coordinates: bool = False
    num_samples: int = 1
    seed: int = 0

    def __post_init__(self):
        if self.num_samples < 1:
            raise ValueError("num_samples must be >= 1")
        if self.seed < 0:
            raise ValueError("seed must be non-negative")


def _is_sampled(est) -> bool:
    return type(est).__name__ == "Sampled" and hasattr(est, "shots")


class GpuEvaluator:
    """Evaluator protocol (ref gradients.py:96-110): ``ev(resolved_circuit, observable, key=None)``."""

    def __init__(self, estimator=Exact()):
        self.estimator = estimator
        self.count = 0

    def __call__(self, circuit, observable, key: tuple = None) -> float:
        from . import sim

        if key is None:
            key = (self.count,)
        self.count += 1
        if _is_sampled(self.estimator):
            seed = derive_seed(self.estimator.seed, *key)
            return sim.sampled_expectation(circuit, observable, self.estimator.shots, seed)
        return sim.expectation(sim.simulate(circuit), observable)


def _require(symbols, bindings):
    miss = [s for s in symbols if s not in bindings]
    if miss:
        raise KeyError(f"missing binding for symbol(s): {', '.join(miss)}")


def _finite(g):
    if not np.all(np.isfinite(g)):
        raise ValueError("gradient has non-finite entries")


# ---------------------------------------------------------------------------
# adjoint
# ---------------------------------------------------------------------------


def adjoint_grad(req: GradRequest) -> GradResult:
    """Exact gradient by the adjoint method (one forward + one backward sweep)."""
    if _is_sampled(req.estimator):
        raise ValueError("the adjoint differentiator needs the Exact estimator")
    c = req.circuit
    obs = as_pauli_sum(req.observable)
    b = normalize_bindings(req.bindings)
    syms = circuit_symbols(c)
    _require(syms, b)
    if not syms:
        return GradResult(np.zeros(0), 0)
    from .ops import expectation_and_gradient

    _, g = expectation_and_gradient([c], syms, np.array([[b[s] for s in syms]], dtype=np.float32), [obs])
    g = np.asarray(g[0], dtype=np.float64)
    _finite(g)
    return GradResult(g, 1)


class Adjoint:
    """Adjoint differentiator engine (``engine(GradRequest) -> GradResult``)."""

    def __call__(self, request: GradRequest) -> GradResult:
        return adjoint_grad(request)


# ---------------------------------------------------------------------------
# parameter shift, batched on the GPU
# ---------------------------------------------------------------------------


def _ps_expand(circuit, bindings, symbols):
    """Per-term rewrite used by PS (ref gradients.py:224-238): symbolic gate j with
    non-identity terms beta_k P_k becomes gates exp(-i eta_jk P_k) with pseudo-symbol
    eta_jk = (coeff_j * theta + const_j) * beta_k.  Returns (circuit, names, values, occ)."""
    index = {s: i for i, s in enumerate(symbols)}
    gates, names, vals, occ = [], [], [], []
    for j, g in enumerate(circuit.gates):
        e = g.exponent
        if e is None or e.symbol is None:
            gates.append(g)
            continue
        gen = as_pauli_sum(g.generator)
        if not all_terms_commute(gen):
            raise ValueError(f"gate {j}: generator terms do not commute, so the parameter-shift "
                             "rule does not apply — use finite_difference_grad instead")
        v = e.coeff * float(bindings[e.symbol]) + e.const
        for t in gen.terms:
            if not t.factors or t.coefficient == 0.0:
                continue  # identity terms: global phase only
            name = f"__ps{j}_{len(names)}"
            gates.append(Gate(tuple(sorted(t.factors)), exponent=ParamExpr(name),
                              generator=PauliSum([PauliString(1.0, t.factors)])))
            names.append(name)
            vals.append(v * t.coefficient)
            occ.append((index[e.symbol], e.coeff * t.coefficient))
    return Circuit(circuit.num_qubits, gates), names, np.array(vals, dtype=np.float64), occ


_PS_CACHE: dict = {}


def _ps_structure(circuit, symbols):
    """Value-independent part of :func:`_ps_expand`: (expanded circuit, pseudo-symbol names,
    spec [(symbol index, coeff, const, beta)] per pseudo-symbol, occ).  base[b, k] =
    (coeff * theta[b, sym] + const) * beta for every row at once.  Cached per circuit object
    (circuits are immutable), so repeated calls reuse one engine binding."""
    key = (id(circuit), tuple(symbols))
    hit = _PS_CACHE.get(key)
    if hit is not None and hit[0] is circuit:
        return hit[1]
    out = _ps_structure_build(circuit, symbols)
    if len(_PS_CACHE) > 256:
        _PS_CACHE.clear()
    _PS_CACHE[key] = (circuit, out)
    return out


def _ps_structure_build(circuit, symbols):
    index = {s: i for i, s in enumerate(symbols)}
    gates, names, spec, occ = [], [], [], []
    for j, g in enumerate(circuit.gates):
        e = g.exponent
        if e is None or e.symbol is None:
            gates.append(g)
            continue
        gen = as_pauli_sum(g.generator)
        if not all_terms_commute(gen):
            raise ValueError(f"gate {j}: generator terms do not commute, so the parameter-shift "
                             "rule does not apply — use finite_difference_grad instead")
        for t in gen.terms:
            if not t.factors or t.coefficient == 0.0:
                continue
            name = f"__ps{j}_{len(names)}"
            gates.append(Gate(tuple(sorted(t.factors)), exponent=ParamExpr(name),
                              generator=PauliSum([PauliString(1.0, t.factors)])))
            names.append(name)
            spec.append((index[e.symbol], float(e.coeff), float(e.const), float(t.coefficient)))
            occ.append((index[e.symbol], e.coeff * t.coefficient))
    return Circuit(circuit.num_qubits, gates), names, spec, occ


def _ps_rows(base, k_count):
    rows = np.repeat(base[None, :], 2 * k_count, axis=0)
    for k in range(k_count):
        rows[2 * k, k] += SHIFT
        rows[2 * k + 1, k] -= SHIFT
    return rows


def _batched_expect(circuit, names, rows, obs, chunk_amps=1 << 31):
    from .ops import expectation

    n = circuit.num_qubits
    per = max(1, chunk_amps >> max(n, 10))
    out = np.empty(rows.shape[0])
    for s in range(0, rows.shape[0], per):
        out[s:s + per] = expectation(circuit, names, rows[s:s + per].astype(np.float32), [obs])[:, 0]
    return out


def parameter_shift_grad(req: GradRequest, evaluator=None) -> GradResult:
    """Exact PS gradient (ref gradients.py:158-165): 2 evaluations per (occurrence, term),
    all executed as one batched GPU launch sequence when no custom evaluator is given."""
    if evaluator is not None or _is_sampled(req.estimator):
        return stochastic_ps_grad(req, StochasticConfig(), evaluator)
    c = req.circuit
    obs = as_pauli_sum(req.observable)
    b = normalize_bindings(req.bindings)
    syms = circuit_symbols(c)
    _require(syms, b)
    if not syms:
        return GradResult(np.zeros(0), 0)
    ec, names, base, occ = _ps_expand(c, b, syms)
    if not names:
        return GradResult(np.zeros(len(syms)), 0)
    f = _batched_expect(ec, names, _ps_rows(base, len(names)), obs)
    grad = np.zeros(len(syms))
    for k, (si, w) in enumerate(occ):
        grad[si] += w * (f[2 * k] - f[2 * k + 1])
    _finite(grad)
    return GradResult(grad, 2 * len(names))


class ParameterShift:
    """Exact parameter-shift engine, GPU-batched (ref graph.py:54-58)."""

    def __call__(self, request: GradRequest) -> GradResult:
        return parameter_shift_grad(request)


def finite_difference_grad(req: GradRequest, scheme: str = CENTRAL, epsilon: float = 1e-4,
                           evaluator=None) -> GradResult:
    """ref gradients.py:113-155; shifted points are batch rows of one execution.
    (In complex64 the central stencil needs epsilon >~ 1e-3 to beat rounding.)"""
    if scheme not in (CENTRAL, FORWARD):
        raise ValueError(f"unknown scheme {scheme!r} (want {CENTRAL!r} or {FORWARD!r})")
    if not epsilon > 0:
        raise ValueError("epsilon must be positive")
    c = req.circuit
    obs = as_pauli_sum(req.observable)
    b = normalize_bindings(req.bindings)
    syms = circuit_symbols(c)
    _require(syms, b)
    if not syms:
        return GradResult(np.zeros(0), 0)
    base = np.array([b[s] for s in syms], dtype=np.float64)
    S = len(syms)
    if evaluator is not None or _is_sampled(req.estimator):
        ev = GpuEvaluator(req.estimator) if evaluator is None else evaluator
        start = ev.count
        from .circuit import resolve

        def f(point):
            return ev(resolve(c, dict(zip(syms, point))), obs)

        g = np.zeros(S)
        if scheme == CENTRAL:
            for k in range(S):
                e = np.zeros(S); e[k] = epsilon
                g[k] = (f(base + e) - f(base - e)) / (2 * epsilon)
        else:
            f0 = f(base)
            for k in range(S):
                e = np.zeros(S); e[k] = epsilon
                g[k] = (f(base + e) - f0) / epsilon
        _finite(g)
        return GradResult(g, ev.count - start)
    eye = np.eye(S) * epsilon
    if scheme == CENTRAL:
        rows = np.concatenate([base + eye, base - eye])
        vals = _batched_expect(c, syms, rows, obs)
        g = (vals[:S] - vals[S:]) / (2 * epsilon)
        n_eval = 2 * S
    else:
        rows = np.concatenate([base[None], base + eye])
        vals = _batched_expect(c, syms, rows, obs)
        g = (vals[1:] - vals[0]) / epsilon
        n_eval = S + 1
    _finite(g)
    return GradResult(g, n_eval)


class FiniteDifference:
    def __init__(self, scheme: str = CENTRAL, epsilon: float = 1e-3):
        if epsilon <= 0:
            raise ValueError("epsilon must be positive")
        self.scheme = scheme
        self.epsilon = float(epsilon)

    def __call__(self, request: GradRequest) -> GradResult:
        return finite_difference_grad(request, self.scheme, self.epsilon)


# ---------------------------------------------------------------------------
# stochastic parameter shift (reference sampling axes, GPU evaluator)
# ---------------------------------------------------------------------------


def _stochastic_walk(occs, cost, cmass, ctot, omass, otot, cfg):
    """The reference's sampling walk (ref gradients.py:263-322), consuming substream(seed, i)
    in exactly its order, WITHOUT evaluating anything: returns the evaluation list
    [(i, occ index, term k, cost term m or -1, weight, counter)] (each entry = the f+ / f-
    pair of keys (i, 0, counter) / (i, 1, counter)) and the degenerate flag."""
    evals = []
    degenerate = False
    for i in range(cfg.num_samples):
        rng = np.random.Generator(np.random.Philox(np.random.SeedSequence(cfg.seed, spawn_key=(i,))))
        counter = 0
        if cfg.sample_coordinates:
            if otot == 0.0:
                degenerate, chosen = True, []
            else:
                pr = omass / otot
                pick = int(rng.choice(len(occs), p=pr))
                chosen = [(pick, 1.0 / pr[pick])]
        else:
            chosen = [(o, 1.0) for o in range(len(occs))]
        for oi, cw in chosen:
            occ = occs[oi]
            terms = occ[4]
            btot = sum(abs(t.coefficient) for t in terms)
            if cfg.sample_generator_terms:
                if btot == 0.0:
                    degenerate = True
                    continue
                k = int(rng.choice(len(terms), p=np.array([abs(t.coefficient) for t in terms]) / btot))
                pairs = [(k, occ[2] * math.copysign(1.0, terms[k].coefficient) * btot)]
            else:
                pairs = [(k, occ[2] * t.coefficient) for k, t in enumerate(terms)]
            for k, w in pairs:
                if w == 0.0:
                    continue
                m = -1
                if cfg.sample_cost_terms:
                    if ctot == 0.0:
                        degenerate = True
                        continue
                    m = int(rng.choice(len(cost), p=cmass / ctot))
                evals.append((i, oi, k, m, cw * w, counter))
                counter += 1
    return evals, degenerate


def stochastic_ps_grad(req: GradRequest, cfg: StochasticConfig, evaluator=None) -> GradResult:
    """ref gradients.py:168-174 / :241-326: Monte-Carlo PS over generator terms, cost terms
    and coordinates with importance weights; substreams keyed exactly as the reference.

    Without a custom ``evaluator`` every shifted evaluation of every sample runs in ONE
    batched launch sequence per observable variant: each shifted circuit is a row of the
    per-term expansion (:func:`_ps_structure`, one pseudo-parameter column per (gate, term)),
    and sampled estimators draw row b with seed derive_seed(est.seed, i, +-, counter) exactly as
    the reference's evaluator does (gradients.py:96-110)."""
    c = req.circuit
    obs = as_pauli_sum(req.observable)
    b = normalize_bindings(req.bindings)
    syms = circuit_symbols(c)
    _require(syms, b)
    if not syms:
        return GradResult(np.zeros(0), 0)
    index = {s: i for i, s in enumerate(syms)}
    occs = []
    for j, g in enumerate(c.gates):
        e = g.exponent
        if e is None or e.symbol is None:
            continue
        gen = as_pauli_sum(g.generator)
        if not all_terms_commute(gen):
            raise ValueError(f"gate {j}: generator terms do not commute, so the parameter-shift "
                             "rule does not apply — use finite_difference_grad instead")
        terms = tuple(t for t in gen.terms if t.factors and t.coefficient != 0.0)
        occs.append((j, index[e.symbol], e.coeff, e.coeff * b[e.symbol] + e.const, terms))
    cost = [t for t in obs.terms if t.factors and t.coefficient != 0.0]
    cmass = np.array([abs(t.coefficient) for t in cost])
    ctot = float(cmass.sum())
    omass = np.array([abs(o[2]) * sum(abs(t.coefficient) for t in o[4]) for o in occs])
    otot = float(omass.sum())
    evals, degenerate = _stochastic_walk(occs, cost, cmass, ctot, omass, otot, cfg)

    def o_eff(m):
        if m < 0:
            return obs
        return PauliSum([cost[m].with_coefficient(math.copysign(1.0, cost[m].coefficient) * ctot)])

    if evaluator is not None:
        # custom evaluator protocol: one call per shifted circuit, in the reference's order
        base = [g.resolved(b) for g in c.gates]

        def shifted(occ, k, delta):
            j, _, _, v, terms = occ
            exp = [Gate(t.support, exponent=ParamExpr(None, 0.0, v * t.coefficient + (delta if kk == k else 0.0)),
                        generator=PauliSum([t.with_coefficient(1.0)])) for kk, t in enumerate(terms)]
            return Circuit(c.num_qubits, base[:j] + exp + base[j + 1:])

        start = evaluator.count
        vals = []
        for i, oi, k, m, w, ctr in evals:
            fp = evaluator(shifted(occs[oi], k, +SHIFT), o_eff(m), key=(i, 0, ctr))
            fm = evaluator(shifted(occs[oi], k, -SHIFT), o_eff(m), key=(i, 1, ctr))
            vals.append((fp, fm))
        n_eval = evaluator.count - start
    else:
        vals = _stochastic_batched(c, syms, b, occs, evals, o_eff, req.estimator)
        n_eval = 2 * len(evals)
    acc = np.zeros(len(syms))
    smp = np.zeros(len(syms))
    cur = 0
    for (i, oi, k, m, w, ctr), (fp, fm) in zip(evals, vals):
        while cur < i:          # the reference adds each sample's vector to acc in order
            acc += smp
            smp = np.zeros(len(syms))
            cur += 1
        smp[occs[oi][1]] += w * (fp - fm)
    while cur < cfg.num_samples:
        acc += smp
        smp = np.zeros(len(syms))
        cur += 1
    g = acc / cfg.num_samples
    _finite(g)
    return GradResult(g, n_eval, degenerate)


def _stochastic_batched(c, syms, b, occs, evals, o_eff, estimator):
    """(f+, f-) for every walk entry: all shifted circuits as rows of the per-term expansion,
    one batched execution per observable variant."""
    from .ops import expectation as op_expectation
    from .ops import sampled_expectation as op_sampled

    if not evals:
        return []
    ec, names, spec, _ = _ps_structure(c, syms)
    theta = np.array([b[s] for s in syms], dtype=np.float64)
    base = np.array([(co * theta[si] + cst) * beta for si, co, cst, beta in spec], dtype=np.float64)
    col0, off = [], 0                      # first pseudo column of each occurrence
    for occ in occs:
        col0.append(off)
        off += len(occ[4])
    R = 2 * len(evals)
    rows = np.repeat(base[None, :], R, axis=0)
    for r, (i, oi, k, m, w, ctr) in enumerate(evals):
        rows[2 * r, col0[oi] + k] += SHIFT
        rows[2 * r + 1, col0[oi] + k] -= SHIFT
    rows32 = rows.astype(np.float32)
    out = np.empty(R)
    by_m: dict = {}
    for r, e in enumerate(evals):
        by_m.setdefault(e[3], []).append(r)
    for m, rs in by_m.items():
        ix = np.array([[2 * r, 2 * r + 1] for r in rs], dtype=np.int64).reshape(-1)
        if _is_sampled(estimator):
            seeds = []
            for r in rs:
                i, _, _, _, _, ctr = evals[r]
                seeds += [derive_seed(estimator.seed, i, 0, ctr), derive_seed(estimator.seed, i, 1, ctr)]
            out[ix] = op_sampled(ec, names, rows32[ix], [o_eff(m)], estimator.shots, seed=seeds)[:, 0]
        else:
            out[ix] = op_expectation(ec, names, rows32[ix], [o_eff(m)])[:, 0]
    return [(out[2 * r], out[2 * r + 1]) for r in range(len(evals))]


class StochasticShift:
    def __init__(self, config: StochasticConfig):
        self.config = config

    def __call__(self, request: GradRequest) -> GradResult:
        return stochastic_ps_grad(request, self.config)
