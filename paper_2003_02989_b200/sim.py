"""Drop-in replacement of the reference's simulation API (qcflow/sim.py), GPU-backed.

Same names, argument meaning, return types and exceptions as ``qcflow.sim``:

=========================  ===============================================  ==========================
function                   reference                                        here
=========================  ===============================================  ==========================
``simulate``               sim.py:139-150 (fused tensordot loop, c128)      tile-pass kernels (c64)
``expectation``            sim.py:203-213                                   fused OBS / Pauli kernels
``batch_execute``          sim.py:275-294 (serial rows)                     one batched launch / topology
``sample``                 sim.py:223-227                                   Philox-exact GPU sampler
``sampled_expectation``    sim.py:245-272                                   per-term substreams on GPU
``run_ops``/``apply_matrix`` sim.py:88-136                                  from-state passes
``pauli_term_values``      sim.py:177-200                                   qf_pauli_expect
``unitary``                sim.py:153-159                                   basis states as batch rows
=========================  ===============================================  ==========================

States are computed in complex64 on the device.  ``StateVector`` keeps the device
tensor (so chained GPU calls never round-trip through the host) and exposes the
reference's complex128 ``amplitudes`` lazily, renormalised in float64 so the
reference's 1e-9 norm invariant (sim.py:50-52) holds for the upcast copy.
"""

from __future__ import annotations

import math
import os
from typing import Sequence

import numpy as np
import torch

from . import gates as gate_lib
from .circuit import Circuit, Gate, circuit_symbols, resolve
from .engine import ENGINE
from .pauli import PauliString, PauliSum, as_pauli_sum, term_masks
from .sampling import bits_from_indices, philox_key, sample_indices

DEFAULT_MAX_QUBITS = 30
NORM_TOL = 1e-9


def max_qubits() -> int:
    """Qubit cap; ``QCFLOW_MAX_QUBITS`` overrides (ref sim.py:27-35).  The default is 30 here
    (2^30 complex64 = 8 GiB of HBM) instead of the reference's CPU-sized 26."""
    raw = os.environ.get("QCFLOW_MAX_QUBITS")
    if raw is None:
        return DEFAULT_MAX_QUBITS
    try:
        return int(raw)
    except ValueError as exc:
        raise ValueError(f"bad QCFLOW_MAX_QUBITS value {raw!r}") from exc


def _check_cap(n: int) -> None:
    cap = max_qubits()
    if n > cap:
        raise MemoryError(f"{n} qubits exceeds the configured cap of {cap} (set QCFLOW_MAX_QUBITS to raise it)")


class StateVector:
    """2^n amplitudes with unit norm (ref sim.py:38-69); device-resident when produced here."""

    __slots__ = ("num_qubits", "_amps", "_dev")

    def __init__(self, num_qubits: int, amplitudes):
        if isinstance(amplitudes, torch.Tensor) and amplitudes.is_cuda:
            dev = amplitudes.reshape(-1)
            if dev.shape[0] != 2 ** num_qubits:
                raise ValueError(f"expected {2 ** num_qubits} amplitudes for {num_qubits} qubits, "
                                 f"got shape {tuple(amplitudes.shape)}")
            object.__setattr__(self, "num_qubits", int(num_qubits))
            object.__setattr__(self, "_amps", None)
            object.__setattr__(self, "_dev", dev)
            return
        a = np.asarray(amplitudes, dtype=np.complex128)
        if a.shape != (2 ** num_qubits,):
            raise ValueError(f"expected {2 ** num_qubits} amplitudes for {num_qubits} qubits, got shape {a.shape}")
        norm = float(np.vdot(a, a).real)
        if abs(norm - 1.0) > NORM_TOL:
            raise ValueError(f"state norm^2 deviates from 1 by {abs(norm - 1.0):.2e}")
        object.__setattr__(self, "num_qubits", int(num_qubits))
        object.__setattr__(self, "_amps", a)
        object.__setattr__(self, "_dev", None)

    def __setattr__(self, key, value):
        raise AttributeError("StateVector is immutable")

    @classmethod
    def zero(cls, num_qubits: int) -> "StateVector":
        a = np.zeros(2 ** num_qubits, dtype=np.complex128)
        a[0] = 1.0
        return cls(num_qubits, a)

    @property
    def amplitudes(self) -> np.ndarray:
        if self._amps is None:
            a = self._dev.cpu().numpy().astype(np.complex128)
            a /= math.sqrt(float(np.vdot(a, a).real))
            a.setflags(write=False)
            object.__setattr__(self, "_amps", a)
        return self._amps

    def device_amplitudes(self, device=None) -> torch.Tensor:
        """complex64 device copy (no host round trip for GPU-produced states)."""
        if self._dev is None:
            dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
            object.__setattr__(self, "_dev", torch.as_tensor(self._amps, dtype=torch.complex64).to(dev))
        return self._dev

    def probabilities(self) -> np.ndarray:
        return np.abs(self.amplitudes) ** 2

    def __repr__(self):
        return f"StateVector(num_qubits={self.num_qubits})"


class SampleBatch:
    """shots x n measured bits, column q = qubit q (ref sim.py:72-85)."""

    __slots__ = ("shots", "bitstrings")

    def __init__(self, shots: int, bitstrings):
        b = np.asarray(bitstrings, dtype=np.uint8)
        if b.ndim != 2 or b.shape[0] != shots:
            raise ValueError("bitstrings must be a shots x n array")
        object.__setattr__(self, "shots", int(shots))
        object.__setattr__(self, "bitstrings", b)

    def __setattr__(self, key, value):
        raise AttributeError("SampleBatch is immutable")


# ---------------------------------------------------------------------------
# simulation
# ---------------------------------------------------------------------------


def _require_concrete(c) -> None:
    if any(g.exponent is not None and g.exponent.symbol is not None for g in c.gates):
        raise KeyError(f"circuit has unresolved symbols: {', '.join(circuit_symbols(c))}")


def simulate(c, fuse_enabled: bool = True) -> StateVector:
    """|0...0> -> U|0...0> on the GPU (ref sim.py:139-150).  ``fuse_enabled`` is accepted for
    signature compatibility; the planner's fusion never changes results beyond rounding."""
    _check_cap(c.num_qubits)
    _require_concrete(c)
    out = ENGINE.bind([c], (), []).execute(_empty_theta(1), want_state=True, want_expect=False)
    return StateVector(c.num_qubits, out["state"][0])


def _empty_theta(rows: int) -> torch.Tensor:
    return torch.zeros((rows, 0), dtype=torch.float32, device=torch.device("cuda", torch.cuda.current_device()))


def simulate_batch(circuits, symbol_names=(), symbol_values=None) -> torch.Tensor:
    """[B, 2^n] complex64 device states of a same-topology batch (no host copies)."""
    circuits = list(circuits)
    vals = _empty_theta(len(circuits)) if symbol_values is None else torch.as_tensor(symbol_values)
    b = ENGINE.bind(circuits, symbol_names, [])
    return b.execute(vals.to(b.device, torch.float32), want_state=True, want_expect=False)["state"]


def _ops_circuit(ops, n):
    gates = [Gate(tuple(tg), matrix=np.asarray(m)) for m, tg in ops]
    return Circuit(n, gates)


def run_ops(amps, ops, num_qubits: int, fuse_enabled: bool = True):
    """Apply a resolved (matrix, targets) list to (a batch of) amplitudes (ref sim.py:122-136).
    numpy in -> complex128 numpy out; CUDA tensor in -> complex64 CUDA tensor out."""
    on_dev = isinstance(amps, torch.Tensor) and amps.is_cuda
    a = amps if on_dev else np.asarray(amps)
    lead = tuple(a.shape[:-1])
    rows = int(np.prod(lead)) if lead else 1
    c = _ops_circuit(ops, num_qubits)
    b = ENGINE.bind([c] * rows, (), [], from_state=True)
    init = a.reshape(rows, -1) if on_dev else torch.as_tensor(np.ascontiguousarray(a.reshape(rows, -1)),
                                                               dtype=torch.complex64)
    out = b.execute(_empty_theta(rows), want_state=True, want_expect=False, initial=init)["state"]
    if on_dev:
        return out.reshape(*lead, -1) if lead else out.reshape(-1)
    res = out.cpu().numpy().astype(np.complex128)
    return res.reshape(*lead, -1) if lead else res.reshape(-1)


def apply_matrix(amps, matrix, targets: Sequence[int], num_qubits: int):
    """One dense 2x2 / 4x4 over ``targets`` (targets[0] = MSB), batch-aware (ref sim.py:88-105)."""
    return run_ops(amps, [(np.asarray(matrix), tuple(targets))], num_qubits)


def unitary(c, bindings=None) -> np.ndarray:
    """Dense 2^n x 2^n unitary (small n; ref sim.py:153-159): basis states as batch rows."""
    cc = resolve(c, bindings)
    dim = 2 ** cc.num_qubits
    eye = np.eye(dim, dtype=np.complex128)
    return run_ops(eye, [(np.asarray(_mat(g)), tuple(g.targets)) for g in cc.gates], cc.num_qubits).T


def _mat(g):
    from .planner import concrete_matrix

    return concrete_matrix(g)


# ---------------------------------------------------------------------------
# expectations
# ---------------------------------------------------------------------------


def _pairwise_sum(values):
    """Deterministic pairwise tree (ref sim.py:162-174)."""
    if not values:
        return 0.0
    work = list(values)
    while len(work) > 1:
        nxt = [work[i] + work[i + 1] for i in range(0, len(work) - 1, 2)]
        if len(work) % 2:
            nxt.append(work[-1])
        work = nxt
    return work[0]


def _term_values_dev(psi: torch.Tensor, n: int, terms) -> torch.Tensor:
    """<psi|P_k|psi> (coefficient 1) for each term, psi [B, 2^n] complex64 -> [B, T] float64."""
    import ctypes as C

    from . import _native as nat

    lib = nat.load()
    B = psi.shape[0]
    n_eff = max(n, 10)
    if n_eff != n:
        full = torch.zeros((B, 1 << n_eff), dtype=torch.complex64, device=psi.device)
        full[:, : 1 << n] = psi
        psi = full
    psi = psi.contiguous()
    xs, zs, ys = zip(*[term_masks(t) for t in terms])
    dev = psi.device
    T = len(terms)
    xm = torch.tensor(np.array(xs, dtype=np.uint32).view(np.int32), device=dev)
    zm = torch.tensor(np.array(zs, dtype=np.uint32).view(np.int32), device=dev)
    ny = torch.tensor(ys, dtype=torch.int32, device=dev)
    cf = torch.ones(T, dtype=torch.float32, device=dev)
    chunks = ((1 << n_eff) + 2047) // 2048
    part = torch.empty((B, T, chunks), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    nat.check(lib.qf_pauli_expect(psi.data_ptr(), n_eff, B, T, xm.data_ptr(), zm.data_ptr(), ny.data_ptr(),
                                  cf.data_ptr(), 0, part.data_ptr(), stream))
    ptr = torch.arange(T + 1, dtype=torch.int32, device=dev)
    lst = torch.arange(T, dtype=torch.int32, device=dev)
    out = torch.empty((B, T), dtype=torch.float64, device=dev)
    nat.check(lib.qf_reduce_slots(part.data_ptr(), B, T, chunks, ptr.data_ptr(), lst.data_ptr(), T, out.data_ptr(),
                                  0, stream))
    return out


def pauli_term_values(amps, term, num_qubits: int):
    """Batch-aware <psi|P|psi> of the coefficient-1 string (ref sim.py:177-200)."""
    on_dev = isinstance(amps, torch.Tensor) and amps.is_cuda
    a = amps if on_dev else torch.as_tensor(np.asarray(amps), dtype=torch.complex64).cuda()
    lead = tuple(a.shape[:-1])
    v = _term_values_dev(a.reshape(-1, a.shape[-1]), num_qubits, [term])[:, 0]
    v = v if on_dev else v.cpu().numpy()
    return v.reshape(lead) if lead else v.reshape(())


def expectation(state: StateVector, obs) -> float:
    """Exact <state|obs|state> (ref sim.py:203-213): identity terms exact, pairwise term sum."""
    obs = as_pauli_sum(obs)
    plain = [t for t in obs.terms if t.factors]
    vals = _term_values_dev(_device_amps(state).reshape(1, -1), state.num_qubits, plain)[0].cpu().numpy() \
        if plain else []
    parts = []
    k = 0
    for t in obs.terms:
        if not t.factors:
            parts.append(t.coefficient)
        else:
            parts.append(t.coefficient * float(vals[k]))
            k += 1
    return float(_pairwise_sum(parts))


def batch_execute(circuits, bindings_matrix, observables) -> np.ndarray:
    """[B, n_obs] exact expectations (ref sim.py:275-294); rows with the same topology run as
    one batched launch; row i binds its values to circuits[i].symbols."""
    observables = [as_pauli_sum(o) for o in observables]
    rows = len(circuits)
    out = np.zeros((rows, len(observables)), dtype=np.float64)
    if rows == 0:
        return out
    groups: dict = {}
    for i, c in enumerate(circuits):
        syms = circuit_symbols(c)
        row = np.atleast_1d(np.asarray(bindings_matrix[i], dtype=np.float64)) if syms else np.zeros(0)
        if len(row) != len(syms):
            raise ValueError(f"row {i}: ragged symbol coverage ({len(row)} values for {len(syms)} symbols)")
        if not np.all(np.isfinite(row)):
            bad = syms[int(np.argmin(np.isfinite(row)))]
            raise ValueError(f"non-finite binding for symbol '{bad}'")
        _check_cap(c.num_qubits)
        from .planner import topology_key

        # the symbol names are part of the key: two circuits of one structure but different
        # symbol names bind different columns of their own rows
        key = (topology_key(c, {s: k for k, s in enumerate(syms)}), tuple(syms))
        groups.setdefault(key, ([], [], syms))
        groups[key][0].append(i)
        groups[key][1].append(row)
    from .ops import expectation as op_expectation

    for idx, vals, syms in groups.values():
        res = op_expectation([circuits[i] for i in idx], syms, np.array(vals, dtype=np.float32).reshape(len(idx), -1),
                             observables)
        out[idx] = res
    return out


# ---------------------------------------------------------------------------
# sampling
# ---------------------------------------------------------------------------


def _device_amps(state) -> torch.Tensor:
    """complex64 device amplitudes of a StateVector of this package, or of any object with the
    reference StateVector's ``num_qubits`` / ``amplitudes`` (ref sim.py:38-69) -- e.g. one a
    user built with qcflow itself before ``install()`` rebound the module."""
    dev_amps = getattr(state, "device_amplitudes", None)
    if dev_amps is not None:
        return dev_amps()
    a = np.asarray(state.amplitudes)
    if a.shape != (2 ** int(state.num_qubits),):
        raise ValueError(f"expected {2 ** int(state.num_qubits)} amplitudes, got shape {a.shape}")
    return torch.as_tensor(a, dtype=torch.complex64).to(torch.device("cuda", torch.cuda.current_device()))


def _padded_dev(state):
    a = _device_amps(state).reshape(1, -1)
    n = state.num_qubits
    n_eff = max(n, 10)
    if n_eff != n:
        full = torch.zeros((1, 1 << n_eff), dtype=torch.complex64, device=a.device)
        full[:, : 1 << n] = a
        a = full
    return a.contiguous(), n_eff


def sample(state: StateVector, shots: int, seed: int) -> SampleBatch:
    """i.i.d. bitstrings from |a_x|^2 with substream(seed) (ref sim.py:223-227)."""
    if shots < 1:
        raise ValueError("shots must be >= 1")
    a, n_eff = _padded_dev(state)
    idx, _ = sample_indices(a, n_eff, shots, [philox_key(seed)])
    return SampleBatch(shots, bits_from_indices(idx[0].cpu().numpy(), state.num_qubits))


def basis_change_gates(term):
    """ref sim.py:230-242."""
    out = []
    for q, p in sorted(term.factors.items()):
        if p == "X":
            out.append(gate_lib.h(q))
        elif p == "Y":
            out.append(gate_lib.zpow(-0.5, q))
            out.append(gate_lib.h(q))
    return out


def sampled_expectation(c, obs, shots_per_term: int, seed: int, fuse_enabled: bool = True) -> float:
    """Shot estimate with per-term basis rotation and substream(seed, k) (ref sim.py:245-272)."""
    if shots_per_term < 1:
        raise ValueError("shots_per_term must be >= 1")
    _check_cap(c.num_qubits)
    _require_concrete(c)
    from .ops import sampled_expectation as op_se

    return float(op_se([c], [], np.zeros((1, 0), dtype=np.float32), [obs], shots_per_term, seed=[seed])[0, 0])
