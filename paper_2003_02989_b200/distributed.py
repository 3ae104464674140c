"""Global-qubit sharding of one circuit across 2^g GPUs (BASELINE.json config 5).

The reference simulates a whole register in one process (qcflow/sim.py:139-150
``simulate``, capped by ``max_qubits`` sim.py:27-35); a 32-qubit complex64 state is
32 GiB, so the B200 build shards it: rank r of 2^g holds the 2^(n-g) amplitudes whose
top g *physical* index bits equal r.  Logical qubits are mapped to physical bits by a
layout that changes only at swaps.

Plan (``plan_segments``, gate-level dependency DAG, diagonal gates commute):
  * a *segment* is every gate that can run without touching a global qubit
    non-diagonally, drained in topological order (a light-cone cut, so a brickwork
    circuit needs a single swap);
  * a *swap* exchanges the g global physical bits with the g top local bits -- one
    all-to-all in which every rank keeps 2^-g of its shard; the qubits brought in are
    the global ones' replacements chosen by fewest remaining non-diagonal gates;
  * the initial layout already places the first swap's qubits on the top local bits, so
    no local permutation is needed unless a plan has swaps with different qubit sets
    (then a ``permute`` step reorders local bits first).

Per rank, a segment becomes an ordinary local circuit on n-g qubits (``localize``):
dense gates are relabelled, diagonal gates touching global qubits are restricted to the
rank's bit values (a Z on a global qubit is a per-rank sign; an all-global diagonal gate
is a relative phase on the shard), and the observable likewise (``localize_observable``),
with identity terms weighted by the shard norm.  Each rank then runs the ordinary engine
(plan-specialised tile passes) with ``from_state`` on its shard in place; per-rank
expectations are summed with one all-reduce.

Exchanges: ``NcclExchange`` (torch.distributed all_to_all_single over NVLink, one
process per GPU) and ``LoopbackExchange`` (all 2^g shards as rows of one device tensor
in one process: the same schedule and arithmetic, the all-to-all becomes a transpose) --
used to check sharded runs against the unsharded one on a single GPU.
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass, field

import numpy as np

from . import planner as pl
from .circuit import Circuit, Gate, circuit_symbols
from .pauli import PauliString, PauliSum, as_pauli_sum


# ---------------------------------------------------------------------------
# plan
# ---------------------------------------------------------------------------


def _gate_is_diag(g) -> bool:
    if g.matrix is not None:
        return pl._concrete_is_diag(g)
    return pl._is_z_only(pl._gate_terms(g))


@dataclass
class Step:
    kind: str                      # "segment" | "swap" | "permute"
    gates: list = field(default_factory=list)      # segment: gate indices in execution order
    perm: list = field(default_factory=list)       # permute: new physical bit of each old local bit
    qubits_in: tuple = ()          # swap: logical qubits that become global
    qubits_out: tuple = ()         # swap: logical qubits that become local


@dataclass
class DistPlan:
    n: int
    g: int
    init_pos: list                 # logical qubit -> physical bit at the start
    steps: list
    pos_before: list               # layout before each step (segments are localised with it)
    final_pos: list

    @property
    def n_loc(self) -> int:
        return self.n - self.g

    @property
    def swaps(self) -> int:
        return sum(s.kind == "swap" for s in self.steps)


def _dependencies(diag, targets):
    last_nd: dict = {}
    diag_since: dict = {}
    preds = []
    for j, (d, tq) in enumerate(zip(diag, targets)):
        p = set()
        for q in tq:
            if q in last_nd:
                p.add(last_nd[q])
            if not d:
                p.update(diag_since.get(q, []))
        preds.append(p)
        for q in tq:
            if d:
                diag_since.setdefault(q, []).append(j)
            else:
                last_nd[q] = j
                diag_since[q] = []
    return preds


def plan_segments(circuit, g: int, keep_local=()) -> DistPlan:
    """``keep_local``: qubits that must end local (observable terms with X/Y on them)."""
    n = circuit.num_qubits
    if g < 0 or g >= n:
        raise ValueError(f"cannot shard {n} qubits over 2^{g} ranks")
    n_loc = n - g
    gates = list(circuit.gates)
    diag = [_gate_is_diag(x) for x in gates]
    targets = [tuple(int(q) for q in x.targets) for x in gates]
    preds = _dependencies(diag, targets)
    succ = [[] for _ in gates]
    npred = [len(p) for p in preds]
    for j, p in enumerate(preds):
        for i in p:
            succ[i].append(j)
    ready = [j for j in range(len(gates)) if npred[j] == 0]
    heapq.heapify(ready)
    done = [False] * len(gates)
    left = len(gates)

    def drain(glob):
        nonlocal left
        taken = []
        while True:
            pick = next((j for j in sorted(ready) if diag[j] or not (set(targets[j]) & glob)), None)
            if pick is None:
                return taken
            ready.remove(pick)
            heapq.heapify(ready)
            done[pick] = True
            left -= 1
            taken.append(pick)
            for s in succ[pick]:
                npred[s] -= 1
                if npred[s] == 0:
                    heapq.heappush(ready, s)

    glob = set(range(n - g, n))
    logical_steps = []
    while True:
        seg = drain(glob)
        logical_steps.append(("segment", seg))
        if left == 0:
            if glob & set(keep_local):
                free = [q for q in range(n) if q not in glob and q not in set(keep_local)]
                if len(free) < g:
                    raise ValueError("observable needs more local qubits than the shard has")
                logical_steps.append(("swap", tuple(sorted(glob)), tuple(free[-g:])))
                logical_steps.append(("segment", []))
            break
        if not seg and logical_steps[:-1] and logical_steps[-2][0] == "swap":
            raise AssertionError("distributed planner made no progress")
        # the next global qubits: fewest remaining non-diagonal gates, avoiding qubits of
        # ready gates (so the following segment makes progress), latest next use first
        remaining = {q: 0 for q in range(n)}
        first_use = {q: len(gates) for q in range(n)}
        for j in range(len(gates)):
            if not done[j] and not diag[j]:
                for q in targets[j]:
                    remaining[q] += 1
                    first_use[q] = min(first_use[q], j)
        busy = {q for j in ready if not diag[j] for q in targets[j]}
        cands = sorted((q for q in range(n) if q not in glob),
                       key=lambda q: (q in busy, remaining[q], -first_use[q], q))
        new = cands[:g]
        logical_steps.append(("swap", tuple(sorted(glob)), tuple(sorted(new))))
        glob = set(new)

    # physical layout: global bits n_loc.., top local bits T = n_loc-g..n_loc-1
    T = list(range(n_loc - g, n_loc))
    G = list(range(n_loc, n))
    first_in = next((s[2] for s in logical_steps if s[0] == "swap"), ())
    pos = [-1] * n
    for i, q in enumerate(range(n - g, n)):
        pos[q] = G[i]
    for i, q in enumerate(first_in):
        pos[q] = T[i]
    free = [b for b in range(n_loc) if b not in set(T[:len(first_in)])]
    for q in range(n):
        if pos[q] < 0:
            pos[q] = free.pop(0)
    init_pos = list(pos)
    steps, pos_before = [], []
    for s in logical_steps:
        if s[0] == "segment":
            pos_before.append(list(pos))
            steps.append(Step("segment", gates=list(s[1])))
            continue
        _, out_q, in_q = s
        if sorted(pos[q] for q in in_q) != T:
            # local permutation: move the incoming qubits onto T (perm: old bit -> new bit)
            perm = list(range(n_loc))
            at = {pos[q]: q for q in range(n) if pos[q] < n_loc}
            movers = [q for q in in_q if pos[q] not in T]
            vacate = [b for b in T if at[b] not in in_q]
            for q, b in zip(movers, vacate):
                a, other = pos[q], at[b]
                perm[a], perm[b] = b, a
                pos[q], pos[other] = b, a
                at[a], at[b] = other, q
            pos_before.append(list(pos))
            steps.append(Step("permute", perm=perm))
        pos_before.append(list(pos))
        steps.append(Step("swap", qubits_in=in_q, qubits_out=out_q))
        phys_in = {pos[q]: q for q in in_q}
        phys_out = {pos[q]: q for q in out_q}
        for i in range(g):
            qi, qo = phys_in[T[i]], phys_out[G[i]]
            pos[qi], pos[qo] = G[i], T[i]
    return DistPlan(n, g, init_pos, steps, pos_before, list(pos))


# ---------------------------------------------------------------------------
# per-rank local circuits / observables
# ---------------------------------------------------------------------------


def _rank_bit(rank: int, phys: int, n_loc: int) -> int:
    return (rank >> (phys - n_loc)) & 1


def localize(circuit, gate_ids, pos, n_loc: int, rank: int) -> Circuit:
    """The segment ``gate_ids`` as rank ``rank``'s circuit on its n_loc local qubits."""
    out = []
    for j in gate_ids:
        gt = circuit.gates[j]
        tq = tuple(int(q) for q in gt.targets)
        ph = tuple(pos[q] for q in tq)
        if all(p < n_loc for p in ph):
            if gt.matrix is not None:
                out.append(Gate(ph, name=gt.name, matrix=gt.matrix))
            else:
                gen = PauliSum([PauliString(t.coefficient, {pos[q]: p for q, p in t.factors.items()})
                                for t in gt.generator.terms])
                out.append(Gate(ph, name=gt.name, exponent=gt.exponent, generator=gen))
            continue
        if not _gate_is_diag(gt):
            raise AssertionError(f"gate {j} acts non-diagonally on a global qubit")
        keep = [i for i, p in enumerate(ph) if p < n_loc]
        loc_t = tuple(ph[i] for i in keep) or (0,)
        if gt.matrix is not None or gt.exponent.symbol is None:
            d = np.diag(pl.concrete_matrix(gt)).astype(np.complex128)
            k = len(tq)
            fixed = 0
            for i, p in enumerate(ph):
                if p >= n_loc and _rank_bit(rank, p, n_loc):
                    fixed |= 1 << (k - 1 - i)       # targets[0] is the MSB of the local index
            if keep:
                sub = []
                for idx in range(1 << len(keep)):
                    full = fixed
                    for jj, i in enumerate(keep):
                        if idx >> (len(keep) - 1 - jj) & 1:
                            full |= 1 << (k - 1 - i)
                    sub.append(d[full])
                out.append(Gate(loc_t, name=gt.name, matrix=np.diag(sub)))
            else:
                out.append(Gate(loc_t, name=gt.name, matrix=np.diag([d[fixed], d[fixed]])))
        else:
            terms = []
            for t in gt.generator.terms:
                sign = 1.0
                f = {}
                for q, p in t.factors.items():
                    if pos[q] >= n_loc:
                        if _rank_bit(rank, pos[q], n_loc):
                            sign = -sign
                    else:
                        f[pos[q]] = p
                terms.append(PauliString(sign * t.coefficient, f))
            out.append(Gate(loc_t, name=gt.name, exponent=gt.exponent, generator=PauliSum(terms)))
    return Circuit(n_loc, out)


def localize_observable(obs, pos, n_loc: int, rank: int) -> PauliSum:
    """Rank ``rank``'s part of a Pauli sum (its expectation on the un-normalised shard;
    the ranks' values add up to the global expectation)."""
    terms = []
    for t in as_pauli_sum(obs).terms:
        sign = 1.0
        f = {}
        for q, p in t.factors.items():
            b = pos[q]
            if b >= n_loc:
                if p != "Z":
                    raise ValueError("observable terms with X/Y on a globally sharded qubit are not supported")
                if _rank_bit(rank, b, n_loc):
                    sign = -sign
            else:
                f[b] = p
        terms.append(PauliString(sign * t.coefficient, f))
    return PauliSum(terms)


# ---------------------------------------------------------------------------
# exchanges
# ---------------------------------------------------------------------------


class LoopbackExchange:
    """All 2^g shards in one process as rows of one tensor; the all-to-all is a transpose."""

    def __init__(self, g: int):
        self.g = g
        self.ranks = list(range(1 << g))

    def swap(self, psi, n_loc: int):
        R = 1 << self.g
        v = psi.reshape(R, R, -1)
        return v.transpose(0, 1).contiguous().reshape(R, -1)

    def allreduce_sum(self, x):
        return x.sum(dim=0, keepdim=True)

    def remote_targets(self, psi):
        """Receive shards for a swap fused into the preceding pass: (peer pointer array on the
        device, rank of row 0, receive tensor)."""
        import torch

        recv = torch.empty_like(psi)
        ptrs = torch.tensor([recv[r].data_ptr() for r in range(recv.shape[0])], dtype=torch.int64,
                            device=psi.device)
        return ptrs, 0, recv

    def remote_done(self):
        pass


class NcclExchange:
    """One process per GPU: rank r owns shard r; swaps are one all_to_all_single
    (torch.distributed, NCCL over NVLink on a B200 box; gloo on CPU in the tests), or -- when
    torch symmetric memory is available -- a store straight into the peers' shards by the
    preceding tile pass (NVLink peer pointers).  The state lives in one of two symmetric
    buffers, rendezvoused ONCE per shape: a fused swap writes into the peers' other buffer,
    which becomes their state (ping-pong), so no swap re-allocates or re-rendezvouses."""

    def __init__(self, g: int, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        world = dist.get_world_size(group)
        if world != 1 << g:
            raise ValueError(f"{world} ranks cannot hold 2^{g} shards")
        self.g = g
        self.ranks = [dist.get_rank(group)]
        # gloo (CPU tests, or several ranks sharing one GPU in the GPU tests) moves host
        # tensors: device shards are staged through host memory, and no symmetric memory
        self.host_staged = dist.get_backend(group) == "gloo"
        self._spare = None
        self._symm = None          # [(buffer, handle, peer-pointer tensor)] x 2, or False
        self._hdl = None

    def _symm_buffers(self, shape, dtype, device):
        import os

        if self.host_staged or os.environ.get("QF_SYMM", "1") in ("0", "", "false"):
            self._symm = False
        if self._symm is False:
            return None
        if self._symm is not None and self._symm[0][0].shape == shape:
            return self._symm
        try:
            import torch
            import torch.distributed._symmetric_memory as symm

            grp = self.dist.group.WORLD if self.group is None else self.group
            bufs = []
            for _ in range(2):
                buf = symm.empty(shape, dtype=dtype, device=device)
                hdl = symm.rendezvous(buf, grp)
                ptrs = torch.tensor([int(p) for p in hdl.buffer_ptrs], dtype=torch.int64, device=device)
                bufs.append((buf, hdl, ptrs))
            self._symm = bufs
        except Exception:
            self._symm = False
            return None
        return self._symm

    def alloc_state(self, rows: int, dim: int, executor):
        """This rank's initial shard, in symmetric memory when available (else None)."""
        if not getattr(executor, "is_cuda", False):
            return None
        torch = executor.torch
        bufs = self._symm_buffers((rows, dim), torch.complex64, executor.device)
        if bufs is None:
            return None
        psi = bufs[0][0]
        psi.zero_()
        return psi

    def swap(self, psi, n_loc: int):
        if self._spare is None or self._spare.shape != psi.shape:
            self._spare = psi.new_empty(psi.shape)
        out = self._spare
        if self.host_staged and psi.is_cuda:
            h_out = out.cpu()
            self.dist.all_to_all_single(_flat(h_out), _flat(psi.cpu()), group=self.group)
            out.copy_(h_out)
        else:
            self.dist.all_to_all_single(_flat(out), _flat(psi), group=self.group)
        self._spare = psi
        return out

    def allreduce_sum(self, x):
        if self.host_staged and x.is_cuda:
            h = x.cpu()
            self.dist.all_reduce(h, group=self.group)
            x.copy_(h)
            return x
        self.dist.all_reduce(x, group=self.group)
        return x

    def remote_targets(self, psi):
        """(peer pointers of every rank's receive shard, this rank, receive tensor) when psi is
        one of the symmetric buffers, else None (plain all-to-all)."""
        bufs = self._symm if self._symm else None
        if not bufs:
            return None
        ptr = psi.data_ptr()
        if ptr == bufs[0][0].data_ptr():
            buf, hdl, ptrs = bufs[1]
        elif ptr == bufs[1][0].data_ptr():
            buf, hdl, ptrs = bufs[0]
        else:
            return None
        self._hdl = hdl
        return ptrs, self.ranks[0], buf

    def remote_done(self):
        self._hdl.barrier()        # stream-ordered: every rank's stores have landed before anyone reads


def _flat(t):
    """1-D real view (chunk c = the top-g local-bit block c of the shard)."""
    import torch

    return torch.view_as_real(t).reshape(-1) if t.is_complex() else t.reshape(-1)


def permute_local_bits(psi, perm, n_loc: int):
    """psi [rows, 2^n_loc]: move local bit a to bit perm[a] (a data-movement pass)."""
    rows = psi.shape[0]
    v = psi.reshape([rows] + [2] * n_loc)          # dim 1 + (n_loc-1-b) holds bit b
    src_dims = [0] * n_loc
    for a in range(n_loc):
        src_dims[n_loc - 1 - perm[a]] = 1 + n_loc - 1 - a
    return v.permute([0] + src_dims).contiguous().reshape(rows, -1)


# ---------------------------------------------------------------------------
# driver
# ---------------------------------------------------------------------------


class EngineExecutor:
    """Runs a batch of per-rank local circuits on the B200 engine, in place on the shards."""

    def __init__(self, device=None):
        import torch

        from .engine import _require_cuda

        self.torch = torch
        self.device = _require_cuda(device)
        self.is_cuda = True

    def zeros(self, rows, dim):
        return self.torch.zeros((rows, dim), dtype=self.torch.complex64, device=self.device)

    def apply(self, circuits, names, values, psi, observables=None, remote=None):
        """observables: None, or one local observable per row (rows differ in signs only).
        remote: (peer pointers, rank of row 0, g) -- the last pass writes the swapped shards
        (only when every row shares one structure and no padding is needed)."""
        from .engine import ENGINE

        torch = self.torch
        theta = torch.as_tensor(np.asarray(values, dtype=np.float32)).to(self.device).reshape(len(circuits), -1)
        if remote is not None:
            b = ENGINE.bind(circuits, names, [], from_state=True, want_state=True, device=self.device)
            b.execute(theta, initial=psi, donate=True, want_state=False, want_expect=False, remote=remote)
            return psi, None
        if observables is None:
            # ranks whose restricted circuits differ in structure (e.g. the sign of a
            # symbolic Z term on a global qubit) run as separate batches
            sym_index = {s: i for i, s in enumerate(names)}
            groups: dict = {}
            for r, c in enumerate(circuits):
                groups.setdefault(pl.topology_key(c, sym_index), []).append(r)
            for rows in groups.values():
                sub = psi if len(rows) == len(circuits) else psi[rows[0]:rows[0] + 1]
                if len(rows) != len(circuits) and len(rows) > 1:
                    sub = psi[rows].contiguous()
                b = ENGINE.bind([circuits[r] for r in rows], names, [], from_state=True, want_state=True,
                                device=self.device)
                st = b.execute(theta[rows], initial=sub, donate=True, want_state=True, want_expect=False)["state"]
                if len(rows) == len(circuits) or len(rows) == 1:
                    if st.data_ptr() != sub.data_ptr():   # registers below the engine minimum are padded
                        sub.copy_(st)
                else:
                    psi[rows] = st
            return psi, None
        if len(circuits) == 1:
            b = ENGINE.bind(circuits, names, observables, from_state=True, norm_identity=True, device=self.device)
            out = b.execute(theta, initial=psi, donate=True)
            return psi, out["expectations"][:, 0]
        vals = []
        for r, (c, o) in enumerate(zip(circuits, observables)):
            b = ENGINE.bind([c], names, [o], from_state=True, norm_identity=True, device=self.device)
            out = b.execute(theta[r:r + 1], initial=psi[r:r + 1], donate=True)
            vals.append(out["expectations"][0, 0])
        return psi, torch.stack(vals)


def _can_fuse(circuits, names, n_loc):
    if n_loc < pl.N_MIN:
        return False
    sym_index = {s: i for i, s in enumerate(names)}
    key = pl.topology_key(circuits[0], sym_index)
    return all(pl.topology_key(c, sym_index) == key for c in circuits[1:])


def run_sharded(circuit, observable, g: int, exchange, executor=None, symbol_names=(), values=None,
                plan: DistPlan | None = None, timer=None, fuse_swaps: bool = True):
    """Expectation of ``observable`` after ``circuit`` on a state sharded over 2^g ranks.

    ``exchange``: LoopbackExchange(g) (all shards here) or NcclExchange(g) (this rank's shard).
    Returns (expectation as float, DistPlan)."""
    keep = sorted({q for t in as_pauli_sum(observable).terms for q, p in t.factors.items() if p != "Z"})
    plan = plan or plan_segments(circuit, g, keep_local=keep)
    executor = executor or EngineExecutor()
    n_loc = plan.n_loc
    ranks = exchange.ranks
    names = list(symbol_names) or circuit_symbols(circuit)
    vals = np.zeros((len(ranks), len(names)), dtype=np.float32)
    if values is not None:
        vals[:] = np.asarray(values, dtype=np.float32).reshape(1, -1)
    alloc = getattr(exchange, "alloc_state", None)
    psi = alloc(len(ranks), 1 << n_loc, executor) if alloc is not None else None
    if psi is None:
        psi = executor.zeros(len(ranks), 1 << n_loc)
    for i, r in enumerate(ranks):
        if r == 0:
            psi[i, 0] = 1.0
    last_seg = max(k for k, s in enumerate(plan.steps) if s.kind == "segment")
    result = None
    skip_swap = False
    for k, (step, pos) in enumerate(zip(plan.steps, plan.pos_before)):
        if timer:
            timer(step.kind, k)
        if step.kind == "segment":
            if not step.gates and k != last_seg:
                continue
            circs = [localize(circuit, step.gates, pos, n_loc, r) for r in ranks]
            if k == last_seg:
                obs = [localize_observable(observable, pos, n_loc, r) for r in ranks]
                psi, result = executor.apply(circs, names, vals, psi, obs)
                continue
            nxt = plan.steps[k + 1] if k + 1 < len(plan.steps) else None
            targets = None
            if (fuse_swaps and nxt is not None and nxt.kind == "swap" and step.gates and
                    isinstance(executor, EngineExecutor) and hasattr(exchange, "remote_targets") and
                    _can_fuse(circs, names, n_loc)):
                targets = exchange.remote_targets(psi)
            if targets is not None:
                # the segment's last pass stores straight into the receive shards (fused swap)
                ptrs, rank0, recv = targets
                executor.apply(circs, names, vals, psi, None, remote=(ptrs.data_ptr(), rank0, g))
                exchange.remote_done()
                psi = recv
                skip_swap = True
            else:
                psi, _ = executor.apply(circs, names, vals, psi, None)
        elif step.kind == "permute":
            psi = permute_local_bits(psi, step.perm, n_loc)
        elif skip_swap:
            skip_swap = False
        else:
            psi = exchange.swap(psi, n_loc)
    if timer:
        timer("end", len(plan.steps))
    tot = exchange.allreduce_sum(result.reshape(-1, 1).clone())
    return float(tot.reshape(-1)[0]), plan
