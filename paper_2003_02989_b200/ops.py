"""TFQ-style batched ops on the B200 engine (the north-star call signatures).

``op(circuits[B], symbol_names[S], symbol_values[B, S], operators[n_obs])``

* ``circuits``: one circuit (broadcast over rows) or a list of B circuits sharing
  a topology (values of concrete gates may differ per row, e.g. data encodings);
* ``symbol_names``: column order of ``symbol_values``;
* ``symbol_values``: numpy / CPU tensor (results come back as numpy, float64) or a
  CUDA tensor (results stay on the device as torch tensors);
* ``operators``: Pauli sums (this package's or the reference's objects).

Reference semantics: qcflow/sim.py ``batch_execute`` (:275-294) for expectations,
``sample`` (:223-227) / ``sampled_expectation`` (:245-272) for the shot-based ops,
and the gradient of ``quantum_backward`` (graph.py:471-513) for the adjoint.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import gates as lib_gates
from . import planner as pl
from .circuit import Circuit
from .engine import ENGINE, UniformBatch
from .pauli import as_pauli_sum
from .sampling import bits_from_indices, derive_seed, philox_key, sample_indices


def _prep(circuits, symbol_values, symbol_names):
    on_dev = isinstance(symbol_values, torch.Tensor) and symbol_values.is_cuda
    if isinstance(symbol_values, torch.Tensor):
        vals = symbol_values
    else:
        vals = torch.as_tensor(np.asarray(symbol_values, dtype=np.float32))
    if vals.ndim == 1:
        vals = vals.reshape(1, -1) if len(symbol_names) else vals.reshape(-1, 0)
    B = int(vals.shape[0])
    if not isinstance(circuits, (list, tuple)):
        circuits = UniformBatch(circuits, B)
    if len(circuits) != B:
        raise ValueError(f"{len(circuits)} circuits for {B} parameter rows")
    if B and vals.shape[1] != len(symbol_names):
        raise ValueError(f"symbol_values has {vals.shape[1]} columns for {len(symbol_names)} symbol names")
    return (circuits if isinstance(circuits, UniformBatch) else list(circuits)), vals, B, on_dev


def _to_dev(vals, dev):
    if vals.is_cuda:
        return vals.to(device=dev, dtype=torch.float32).contiguous()
    if vals.dtype != torch.float32:
        vals = vals.to(torch.float32)
    return vals.to(dev, non_blocking=vals.is_pinned()).contiguous()


def _out(t, on_dev):
    return t if on_dev else t.cpu().numpy()


def _outs(ts, on_dev):
    """Several device results to the host with ONE stream synchronisation: asynchronous
    copies into pinned buffers (torch's caching host allocator), then a single sync."""
    if on_dev:
        return tuple(ts)
    if not all(t.is_cuda and t.device == ts[0].device for t in ts) or len(devices()) > 1:
        return tuple(t.cpu().numpy() for t in ts)
    hs = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in ts]
    for h, t in zip(hs, ts):
        h.copy_(t, non_blocking=True)
    torch.cuda.current_stream(ts[0].device).synchronize()
    return tuple(h.numpy() for h in hs)


# ---------------------------------------------------------------------------
# row partitioning: one launch sequence per (topology, device)
# ---------------------------------------------------------------------------

_DEVICES: list | None = None
# a part must move at least this many amplitudes per device before a batch is split
SPLIT_MIN_AMPS = 1 << 22


def set_devices(devices) -> None:
    """Devices every ``ops.*`` call splits its rows over (one host process
    drives all GPUs; rows are independent, so the split needs no collective).  ``None``
    restores the default: ``QF_DEVICES`` ("all" or "0,1,...") or the current device."""
    global _DEVICES
    _DEVICES = None if devices is None else [torch.device("cuda", int(getattr(d, "index", d) or 0))
                                             for d in devices]


def devices() -> list:
    if _DEVICES is not None:
        return list(_DEVICES)
    from .engine import _require_cuda

    env = os.environ.get("QF_DEVICES", "")
    if env:
        _require_cuda(None)
        ids = range(torch.cuda.device_count()) if env == "all" else [int(x) for x in env.split(",") if x]
        return [torch.device("cuda", i) for i in ids]
    return [_require_cuda(None)]


def _subset(circuits, idx):
    if isinstance(circuits, UniformBatch):
        return UniformBatch(circuits.circuit, len(idx))
    return [circuits[i] for i in idx]


def topology_groups(circuits, symbol_names) -> list:
    """Row-index arrays of the rows that share one topology (first-row order), so a batch
    whose rows differ in structure -- e.g. the reference QCNN app's per-row data circuits
    (apps/qcnn.py task_circuits) -- runs as one launch sequence per topology."""
    from .planner import topology_key

    index = {s: i for i, s in enumerate(symbol_names)}
    keys: dict = {}
    memo: dict = {}
    for b, c in enumerate(circuits):
        k = memo.get(id(c))
        if k is None:
            try:
                k = topology_key(c, index)
            except KeyError as exc:
                raise KeyError(f"missing binding for symbol {exc.args[0]!r}") from None
            memo[id(c)] = k
        keys.setdefault(k, []).append(b)
    return [np.asarray(v, dtype=np.int64) for v in keys.values()]


def _split(rows: int, n_amps: int, n_dev: int) -> list:
    if n_dev <= 1 or rows < 2:
        return [(0, rows)]
    k = int(min(n_dev, rows, max(1, (rows * n_amps) // SPLIT_MIN_AMPS)))
    base, extra = divmod(rows, k)
    out, s = [], 0
    for r in range(k):
        e = s + base + (1 if r < extra else 0)
        out.append((s, e))
        s = e
    return out


def _run(circuits, symbol_names, vals, observables=(), *, want_grad=False, want_state=False,
         want_expect=True, upstream=None, post=None, keys=("expectations",)):
    """Bind + execute ``circuits`` (B rows) split by topology and over :func:`devices`.
    ``post(out, bound, rows)`` (optional) maps one part's outputs, on its device, to the
    tensors to return; row-ordered results land on the device of ``vals`` (or the first
    device).  Launches on different devices overlap: each part is issued asynchronously
    on its device's current stream before any result is gathered."""
    B = len(circuits)
    devs = devices()
    n = circuits[0].num_qubits
    groups = [None]
    while True:
        parts = []
        for g in groups:
            rows = B if g is None else len(g)
            for a, b in _split(rows, 1 << max(n, 10), len(devs)):
                idx = None if (g is None and a == 0 and b == B) else \
                    (np.arange(a, b, dtype=np.int64) if g is None else g[a:b])
                parts.append(idx)
        outs = []
        try:
            for j, idx in enumerate(parts):
                d = devs[j % len(devs)] if len(devs) > 1 else devs[0]
                sub = circuits if idx is None else _subset(circuits, idx)
                with torch.cuda.device(d):
                    bound = ENGINE.bind(sub, symbol_names, observables, want_grad=want_grad, device=d,
                                        want_state=want_state)
                    v = vals if idx is None else vals[torch.as_tensor(idx, device=vals.device)]
                    up = None
                    if upstream is not None:
                        if idx is None:
                            up = upstream
                        elif isinstance(upstream, torch.Tensor):
                            up = upstream[torch.as_tensor(idx, device=upstream.device)]
                        else:
                            up = np.asarray(upstream)[idx]
                    out = bound.execute(_to_dev(v, d), upstream=up, want_grad=want_grad, want_state=want_state,
                                        want_expect=want_expect)
                    if post is not None:
                        out = post(out, bound, idx)
                outs.append((idx, d, out))
            break
        except pl.TopologyMismatch:
            if groups != [None]:
                raise
            groups = topology_groups(circuits, symbol_names)
    home = vals.device if vals.is_cuda else devs[0]
    if len(outs) == 1 and outs[0][0] is None and outs[0][1] == home:
        return outs[0][2]
    res = {}
    for key in keys:
        first = outs[0][2][key]
        full = torch.empty((B,) + tuple(first.shape[1:]), dtype=first.dtype, device=home)
        for idx, d, out in outs:
            part = out[key].to(home, non_blocking=True)
            if idx is None:
                full.copy_(part)
            else:
                full[torch.as_tensor(idx, device=home)] = part
        res[key] = full
    return res


def expectation(circuits, symbol_names, symbol_values, operators):
    """[B, n_obs] exact expectations (float64)."""
    circuits, vals, B, on_dev = _prep(circuits, symbol_values, symbol_names)
    ops = [as_pauli_sum(o) for o in operators]
    if B == 0:
        return np.zeros((0, len(ops)))
    out = _run(circuits, symbol_names, vals, ops)
    return _out(out["expectations"], on_dev)


def expectation_and_gradient(circuits, symbol_names, symbol_values, operators, upstream=None):
    """(expectations [B, n_obs], d<sum_k upstream[b,k] O_k>/d symbol_values [B, S]) via the
    adjoint method (one forward + one backward sweep per batch)."""
    circuits, vals, B, on_dev = _prep(circuits, symbol_values, symbol_names)
    ops = [as_pauli_sum(o) for o in operators]
    if B == 0:
        return np.zeros((0, len(ops))), np.zeros((0, len(symbol_names)))
    out = _run(circuits, symbol_names, vals, ops, want_grad=True, upstream=upstream,
               keys=("expectations", "grad"))
    return _outs((out["expectations"], out["grad"]), on_dev)


def expectation_and_ps_gradient(circuits, symbol_names, symbol_values, operators, upstream=None,
                                chunk_amps: int = 1 << 31):
    """As :func:`expectation_and_gradient`, with the reference's exact parameter-shift rule
    (ref gradients.py:158-165, 241-326: 2 evaluations per (occurrence, generator term),
    shift pi/4, no 1/2 factor) instead of the adjoint sweep.  All B rows x 2*sum K shifted
    circuits run as batched engine launches (``chunk_amps`` amplitudes per launch)."""
    from . import gradients as gr
    from .circuit import circuit_symbols

    circuits, vals, B, on_dev = _prep(circuits, symbol_values, symbol_names)
    ops = [as_pauli_sum(o) for o in operators]
    S = len(symbol_names)
    if B == 0:
        return np.zeros((0, len(ops))), np.zeros((0, S))
    if not isinstance(circuits, UniformBatch) and any(c is not circuits[0] for c in circuits):
        groups_t = topology_groups(circuits, symbol_names)
        if len(groups_t) > 1:   # one batched parameter-shift sweep per topology
            e_all = np.zeros((B, len(ops)))
            g_all = np.zeros((B, S))
            up_np = None if upstream is None else np.asarray(upstream, dtype=np.float64).reshape(B, -1)
            vals_h = vals.detach().cpu()
            for g in groups_t:
                e_g, g_g = expectation_and_ps_gradient([circuits[i] for i in g], symbol_names,
                                                       vals_h[torch.as_tensor(g)], ops,
                                                       None if up_np is None else up_np[g], chunk_amps)
                e_all[g], g_all[g] = e_g, g_g
            if on_dev:
                return torch.as_tensor(e_all, device=vals.device), torch.as_tensor(g_all, device=vals.device)
            return e_all, g_all
    vals_np = vals.detach().cpu().numpy().astype(np.float32).astype(np.float64).reshape(B, -1)
    col = {s: i for i, s in enumerate(symbol_names)}
    up = np.ones((B, len(ops))) if upstream is None else np.asarray(upstream, dtype=np.float64).reshape(B, -1)
    # rows sharing one circuit object share one expanded circuit (values differ only)
    groups: dict = {}
    for b, c in enumerate(circuits):
        groups.setdefault(id(c), []).append(b)
    structs = {}
    names0 = None
    for key, bs in groups.items():
        c = circuits[bs[0]]
        syms_c = circuit_symbols(c)
        ec, names, spec, occ = gr._ps_structure(c, syms_c)
        if names0 is None:
            names0 = names
        elif names != names0:
            raise ValueError("all circuits of a batch must share one topology")
        cols = np.array([col[syms_c[si]] for si, _, _, _ in spec], dtype=np.int64)
        coeff = np.array([x[1] for x in spec]); const = np.array([x[2] for x in spec])
        beta = np.array([x[3] for x in spec])
        base = (coeff[None, :] * vals_np[bs][:, cols] + const[None, :]) * beta[None, :] if spec else None
        structs[key] = (ec, base, [(col[syms_c[si]], w) for si, w in occ])
    K = len(names0 or [])
    dev = _device()
    grad_d = None
    if K:
        # every host table goes to the device before the first launch (a pageable host->device
        # copy waits for the stream, so a copy between launches idles the GPU)
        base_all = np.empty((B, K))
        # gradient = d @ W per group: W[k, s] = sum of the occurrence weights of pseudo-symbol k
        Ws = {}
        for key, bs in groups.items():
            base_all[bs] = structs[key][1]
            W = np.zeros((K, S))
            for k, (si, w) in enumerate(structs[key][2]):
                W[k, si] += w
            Ws[key] = torch.as_tensor(W, device=dev)
        upd = torch.as_tensor(up, dtype=torch.float64, device=dev)
        rows = torch.as_tensor(base_all, dtype=torch.float64, device=dev)[:, None, :].repeat(1, 2 * K, 1)
        kk = torch.arange(K, device=dev)
        rows[:, 2 * kk, kk] += gr.SHIFT
        rows[:, 2 * kk + 1, kk] -= gr.SHIFT
        allrows = rows.reshape(B * 2 * K, K).to(torch.float32)
        n_eff = max(circuits[0].num_qubits, 10)
        per = max(1, chunk_amps >> n_eff)
        f = torch.empty((B * 2 * K, len(ops)), dtype=torch.float64, device=dev)
        for s0 in range(0, allrows.shape[0], per):
            s1 = min(s0 + per, allrows.shape[0])
            if len(groups) == 1:
                cs = structs[next(iter(groups))][0]
            else:
                cs = [structs[id(circuits[r // (2 * K)])][0] for r in range(s0, s1)]
            f[s0:s1] = expectation(cs, names0, allrows[s0:s1], ops)
        f = (f.reshape(B, K, 2, len(ops)) * upd[:, None, None, :]).sum(dim=3)
        d = f[:, :, 0] - f[:, :, 1]                                       # [B, K]
        if len(groups) == 1:
            grad_d = d @ Ws[next(iter(groups))]
        else:
            grad_d = torch.zeros((B, S), dtype=torch.float64, device=dev)
            for key, bs in groups.items():
                ix = torch.as_tensor(bs, device=dev)
                grad_d[ix] = d[ix] @ Ws[key]
    e0 = expectation(circuits, symbol_names, vals, ops)
    if grad_d is None:
        grad_d = torch.zeros((B, S), dtype=torch.float64, device=dev)
    if on_dev:
        dev = vals.device
        return torch.as_tensor(e0, device=dev), grad_d.to(dev)
    return (e0.detach().cpu().numpy() if isinstance(e0, torch.Tensor) else e0), grad_d.cpu().numpy()


def state(circuits, symbol_names, symbol_values):
    """[B, 2^n] complex64 final states (device tensor; numpy complex64 for host inputs)."""
    circuits, vals, B, on_dev = _prep(circuits, symbol_values, symbol_names)
    out = _run(circuits, symbol_names, vals, want_state=True, want_expect=False, keys=("state",))
    return _out(out["state"], on_dev)


def _device():
    from .engine import _require_cuda

    return _require_cuda(None)


def _row_seeds(seed, B):
    if isinstance(seed, (list, tuple, np.ndarray)):
        if len(seed) != B:
            raise ValueError("need one seed per row")
        return [int(s) for s in seed]
    return [derive_seed(int(seed), b) for b in range(B)]


def _state_for_sampling(out, bound):
    n, n_eff = bound.plan.n, bound.plan.n_eff
    return out["state"] if n_eff == n else _padded(out["state"], n_eff), n_eff


def sample(circuits, symbol_names, symbol_values, repetitions: int, seed=0):
    """Bitstrings [B, repetitions, n] uint8 (column q = qubit q); row b draws with
    substream(seed_b) where seed_b = seed[b] or derive_seed(seed, b) (ref sim.py:223-227)."""
    if repetitions < 1:
        raise ValueError("shots must be >= 1")
    circuits, vals, B, on_dev = _prep(circuits, symbol_values, symbol_names)
    seeds = _row_seeds(seed, B)

    def draw(out, bound, idx):
        psi, n_eff = _state_for_sampling(out, bound)
        rows = range(B) if idx is None else idx
        idx_t, _ = sample_indices(psi, n_eff, repetitions, [philox_key(seeds[r]) for r in rows])
        return {"idx": idx_t}

    out = _run(circuits, symbol_names, vals, want_state=True, want_expect=False, post=draw, keys=("idx",))
    return bits_from_indices(out["idx"].cpu().numpy(), circuits[0].num_qubits)


def _padded(st, n_eff):
    B, d = st.shape
    full = torch.zeros((B, 1 << n_eff), dtype=st.dtype, device=st.device)
    full[:, :d] = st
    return full


def _basis_gates(term):
    """ref sim.py:230-242: H for X; Z**-0.5 then H for Y."""
    out = []
    for q, p in sorted(term.factors.items()):
        if p == "X":
            out.append(lib_gates.h(q))
        elif p == "Y":
            out.append(lib_gates.zpow(-0.5, q))
            out.append(lib_gates.h(q))
    return out


def sampled_expectation(circuits, symbol_names, symbol_values, operators, repetitions: int, seed=0):
    """[B, n_obs] shot estimates with the reference's per-term semantics: term k of an
    operator is measured in its own rotated basis with substream(seed_b, k)
    (ref sim.py:245-272; seed_b as in :func:`sample`).  Terms sharing a basis rotation
    share one simulated state; all terms of a basis are drawn by one sampler launch."""
    if repetitions < 1:
        raise ValueError("shots_per_term must be >= 1")
    circuits, vals, B, on_dev = _prep(circuits, symbol_values, symbol_names)
    seeds = _row_seeds(seed, B)
    ops = [as_pauli_sum(o) for o in operators]
    res = np.zeros((B, len(ops)))
    # group (op, term) by basis rotation signature
    groups: dict = {}
    for oi, o in enumerate(ops):
        parts = []
        for k, t in enumerate(o.terms):
            if not t.factors:
                parts.append(("ident", t.coefficient))
                continue
            sig = tuple(sorted((q, p) for q, p in t.factors.items() if p != "Z"))
            groups.setdefault(sig, []).append((oi, k, t))
            parts.append(("term", k))
        ops[oi] = (o, parts)
    values_per_term: dict = {}
    for sig, members in groups.items():
        extra = _basis_gates(members[0][2].__class__(1.0, dict(sig))) if sig else []
        if extra:
            rot = [Circuit(c.num_qubits, tuple(c.gates) + tuple(extra)) for c in
                   ([circuits.circuit] if isinstance(circuits, UniformBatch) else circuits)]
            rot = UniformBatch(rot[0], B) if isinstance(circuits, UniformBatch) else rot
        else:
            rot = circuits
        # every term of this basis draws from the same state: the state is repeated once per
        # term as sampler rows (keys substream(seed_b, k)), one launch for all of them
        ks = sorted({k for _, k, _ in members})

        def draw(out, bound, idx, ks=ks):
            psi, n_eff = _state_for_sampling(out, bound)
            rows = list(range(B)) if idx is None else list(idx)
            keys = [philox_key(seeds[r], k) for r in rows for k in ks]
            idx_t, _ = sample_indices(psi.contiguous(), n_eff, repetitions, keys, keys_per_row=len(ks))
            return {"idx": idx_t.reshape(len(rows), len(ks), repetitions)}

        out = _run(rot, symbol_names, vals, want_state=True, want_expect=False, post=draw, keys=("idx",))
        idx_all = out["idx"].cpu().numpy()                      # [B, len(ks), shots]
        for oi, k, t in members:
            idx = idx_all[:, ks.index(k), :]
            mask = 0
            for q in t.factors:
                mask |= 1 << q
            par = np.zeros(idx.shape, dtype=np.int64)
            m = idx & mask
            while np.any(m):
                par ^= m & 1
                m = m >> 1
            eig = 1.0 - 2.0 * par
            values_per_term[(oi, k)] = t.coefficient * eig.mean(axis=1)
    for oi, (o, parts) in enumerate(ops):
        contrib = []
        for kind, x in parts:
            contrib.append(np.full(B, x) if kind == "ident" else values_per_term[(oi, x)])
        res[:, oi] = _pairwise(contrib) if contrib else 0.0
    return res


def _pairwise(values):
    """Deterministic pairwise tree (ref sim.py:162-174), applied elementwise over rows."""
    work = list(values)
    while len(work) > 1:
        nxt = [work[i] + work[i + 1] for i in range(0, len(work) - 1, 2)]
        if len(work) % 2:
            nxt.append(work[-1])
        work = nxt
    return work[0]
