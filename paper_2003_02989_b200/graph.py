"""Layer-level batched entry points (ref qcflow/graph.py:443-549) on the GPU engine.

``quantum_forward(node, param_batch)`` and ``quantum_backward(node, param_batch,
upstream)`` accept the reference's quantum nodes (``PQC`` / ``ControlledPQC`` --
anything exposing ``model_circuit``, ``observables``, ``symbols``, ``estimator``,
``differentiator``, ``_data_batch``, ``_combined``, ``_next_call``) and run each
batch as ONE launch sequence: row b is data circuit b followed by the model
circuit bound to parameter row b.  Exact estimators use the adjoint method for the
backward pass (the vector-Jacobian product of graph.py:471-513 without a per-row
loop); sampled estimators keep the reference's per-row seeds
``derive_seed(seed, call_id, b, k)`` (graph.py:463-467).
"""

from __future__ import annotations

import numpy as np

from .gradients import Adjoint, FiniteDifference, GradRequest, ParameterShift, Sampled, finite_difference_grad
from .ops import expectation, expectation_and_gradient, sampled_expectation
from .sampling import derive_seed


def _check(node, param_batch):
    pb = np.atleast_2d(np.asarray(param_batch, dtype=np.float64))
    want = len(node.symbols)
    if pb.ndim != 2 or pb.shape[1] != want:
        raise ValueError(f"{node.name}: symbol mismatch — parameter rows have width {pb.shape[-1]} "
                         f"but the model circuit has {want} symbols")
    return pb


def _is_exact(est) -> bool:
    return type(est).__name__ == "Exact"


def quantum_forward(node, param_batch) -> np.ndarray:
    pb = _check(node, param_batch)
    rows = pb.shape[0]
    data = node._data_batch(rows)
    call_id = node._next_call()
    circuits = [node._combined(d) for d in data]
    syms = list(node.symbols)
    if _is_exact(node.estimator):
        return np.asarray(expectation(circuits, syms, pb.astype(np.float32), node.observables), dtype=np.float64)
    out = np.zeros((rows, len(node.observables)))
    est = node.estimator
    for k, obs in enumerate(node.observables):
        seeds = [derive_seed(est.seed, call_id, b, k) for b in range(rows)]
        out[:, k] = sampled_expectation(circuits, syms, pb.astype(np.float32), [obs], est.shots, seed=seeds)[:, 0]
    return out


def quantum_backward(node, param_batch, upstream) -> np.ndarray:
    pb = _check(node, param_batch)
    rows, width = pb.shape
    up = np.asarray(upstream, dtype=np.float64)
    if up.shape != (rows, len(node.observables)):
        raise ValueError(f"{node.name}: upstream shape {up.shape} != ({rows}, {len(node.observables)})")
    if width == 0:
        return np.zeros((rows, 0))
    data = node._data_batch(rows)
    call_id = node._next_call()
    circuits = [node._combined(d) for d in data]
    syms = list(node.symbols)
    diff = node.differentiator
    name = type(diff).__name__
    if _is_exact(node.estimator) and name in ("Adjoint", "ParameterShift"):
        _, g = expectation_and_gradient(circuits, syms, pb.astype(np.float32), node.observables, upstream=up)
        return np.asarray(g, dtype=np.float64)
    # generic path: one weighted-observable request per row (ref graph.py:497-512)
    out = np.zeros((rows, width))
    for b in range(rows):
        w = up[b]
        if not w.any():
            continue
        weighted = None
        for k, obs in enumerate(node.observables):
            if w[k] != 0.0:
                term = obs * float(w[k])
                weighted = term if weighted is None else weighted + term
        est = node.estimator
        if not _is_exact(est):
            est = type(est)(est.shots, derive_seed(est.seed, call_id, b))
        req = GradRequest(circuits[b], weighted, dict(zip(syms, pb[b])), est)
        out[b] = diff(req).gradient
    return out


__all__ = ["quantum_forward", "quantum_backward", "Adjoint", "ParameterShift", "FiniteDifference",
           "finite_difference_grad", "Sampled"]
