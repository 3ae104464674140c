"""Topology planner: circuit -> fused ops -> tile passes -> register stages -> device program.

This replaces the per-row host work of the reference (``resolve`` + ``gate_matrix`` +
``fuse_resolved`` per row and per evaluation, qcflow/sim.py:116-136,
fusion.py:78-176) with a plan that is built ONCE per circuit topology and shared
by every batch row; the per-row numbers (matrices, phase angles) are produced on
the GPU by ``qf_build_ops`` from the ``[batch, n_symbols]`` value matrix.

Fusion here differs from the reference's qsim-style pass in what it is optimised
for, not in results: 1q runs are merged, 1q gates fold into neighbouring dense
2q gates, and every diagonal gate (Z-type generators, CZ, S, T, ...) becomes a
term of a *phase polynomial* ``exp(-i sum_k theta_k Z_{m_k})`` that the kernel
evaluates from the amplitude index without moving data.  Adjoint programs keep
every symbolic gate separate (a gradient slot each) and only fuse fixed gates.

Geometry (see csrc/qf_pass.cu): a pass owns a tile of L qubits that always
contains qubits 0..4 (coalesced 256-byte warp accesses); inside a pass, stages
choose which R tile bits live in registers; dense ops must sit on register bits.
"""

from __future__ import annotations

import heapq
import math
from dataclasses import dataclass, field

import numpy as np

from .circuit import generator_matrix, gate_matrix
from .pauli import term_masks

N_MIN = 10          # smaller registers are padded (extra qubits stay |0>)
LANE_Q = 4          # qubits 0..3 are always lane bits at load/store (128-byte runs)
FWD_L, FWD_R = 12, 5   # 4 CTAs/SM x 128 threads at 128 registers: fastest measured (tools/sweep.sh)
ADJ_L, ADJ_R = 12, 4



def geometry(adjoint: bool) -> tuple:
    """(L, R) of the tile passes; QF_GEOM_FWD / QF_GEOM_ADJ="L,R" override (experiments;
    only the plan-specialised kernels support geometries other than the defaults)."""
    import os

    env = os.environ.get("QF_GEOM_ADJ" if adjoint else "QF_GEOM_FWD")
    if env:
        L, R = (int(x) for x in env.split(","))
        return L, R
    return (ADJ_L, ADJ_R) if adjoint else (FWD_L, FWD_R)


OP_DENSE1, OP_DENSE2, OP_DIAG, OP_OBS = 1, 2, 3, 4
CLS_GENERAL, CLS_XLIKE, CLS_REAL = 0, 1, 2   # dense 1q matrix structure classes
CLS_NX, CLS_NY = 3, 4                       # Pauli-frame normalised X / Y rotations: [[1, -i tau], [-i tau, 1]] / [[1, -tau], [tau, 1]]
CLS_NP = 5                                  # normalised two-qubit Pauli-string rotation I - i tau P0 P1
EV_NX, EV_NY, EV_ABS1, EV_ABS2, EV_DIAG, EV_OBS, EV_NP = 1, 2, 3, 4, 5, 6, 7   # frame-walk events
EV_PASS = 8    # pass boundary: forward records the stored state's scale, adjoint reloads it
PAULI_CODE = {"X": 1, "Y": 2, "Z": 3}
EV_INTS = 8
GK_MATRIX, GK_X, GK_Y, GK_Z = 0, 1, 2, 3     # adjoint generator kinds (GK_P: two-qubit Pauli string)
GK_P = 4
INIT_LOAD, INIT_ZERO, INIT_PRODUCT, INIT_LOAD_PSI = 0, 1, 2, 3

STAGE_INTS, OP_INTS, PASS_INTS = 64, 16, 128
# op row: 0 kind, 1-2 register slots, 3 matrix offset, 4-6 term range / subset table, 7 slot,
# 8 generator offset, 9 class, 10 generator kind, 11 frame x column, 12 Pauli-string code,
# 13 block dimension, 14 merged-slot role (1 head, 2 member), 15 lane op: 1 + thread bit (0: none)
# measured: two extra live accumulators push the 128-register adjoint kernels into spills
# (SASS: +35 MOV per amplitude), so merging is off by default
MERGE_SLOTS = __import__("os").environ.get("QF_MERGE_SLOTS", "0") not in ("0", "", "false")


def swizzle(l: int) -> int:
    """GF(2)-linear smem swizzle: low 4 bits ^= bits 4-7 ^ 8-11 ^ 12-15."""
    return l ^ ((l >> 4) & 15) ^ ((l >> 8) & 15) ^ ((l >> 12) & 15)


# ---------------------------------------------------------------------------
# gate analysis
# ---------------------------------------------------------------------------


@dataclass
class GateInfo:
    index: int
    targets: tuple
    symbolic: bool
    diag: bool
    sym: int = -1          # symbol column
    coeff: float = 0.0
    const: float = 0.0
    terms: list = field(default_factory=list)   # [(factors dict, coeff)] generator terms
    gen: int = -1          # index in the generator table (symbolic gates)
    fixed: int = -1        # index in the fixed-matrix table (concrete dense gates)
    const_col: int = -1    # first constant-angle column (concrete diagonal gates)
    cls: int = CLS_GENERAL  # dense 1q structure class (same for every row of a topology)
    axis: str = ""          # "X" / "Y": a 1q rotation exp(-i v P) (+ global phase) -> frame-normalisable
    pstring: tuple = ()     # 2q rotation exp(-i v beta P0 P1) (+ identity): ((q0, letter), (q1, letter))


def _is_z_only(terms) -> bool:
    return all(all(p == "Z" for p in f.values()) for f, _ in terms)


def _gate_terms(g):
    return [(dict(t.factors), float(t.coefficient)) for t in g.generator.terms]


def _symbolic_class(terms, targets) -> int:
    if len(targets) != 1:
        return CLS_GENERAL
    letters = {p for f, c in terms for p in f.values()}
    has_ident = any(not f and c != 0.0 for f, c in terms)
    if has_ident or len(letters) != 1:
        return CLS_GENERAL
    return {"X": CLS_XLIKE, "Y": CLS_REAL}.get(letters.pop(), CLS_GENERAL)


def _rotation_axis(terms, targets) -> str:
    """"X"/"Y" when the generator is a single-qubit Pauli (plus an identity term)."""
    if len(targets) != 1:
        return ""
    letters = {p for f, c in terms for p in f.values() if c != 0.0}
    if any(len(f) > 1 for f, _ in terms) or len(letters) != 1:
        return ""
    a = letters.pop()
    return a if a in ("X", "Y") else ""


def _pauli_string(terms, targets) -> tuple:
    """((q0, P0), (q1, P1)) when the generator is one two-qubit, non-diagonal Pauli string
    (plus an identity term)."""
    if len(targets) != 2:
        return ()
    plain = [(f, c) for f, c in terms if f and c != 0.0]
    if len(plain) != 1 or set(plain[0][0]) != set(targets):
        return ()
    f = plain[0][0]
    if all(p == "Z" for p in f.values()):
        return ()
    return tuple((q, f[q]) for q in targets)


def _matrix_class(m) -> int:
    if m.shape[0] != 2:
        return CLS_GENERAL
    if np.all(m.imag == 0):
        return CLS_REAL
    if m[0, 0].imag == 0 and m[1, 1].imag == 0 and m[0, 1].real == 0 and m[1, 0].real == 0:
        return CLS_XLIKE
    return CLS_GENERAL


def _concrete_class(g) -> int:
    return _matrix_class(concrete_matrix(g))


def topology_key(circuit, symbol_index) -> tuple:
    """Structure that must match for rows to share one plan (values may differ)."""
    out = [circuit.num_qubits]
    for g in circuit.gates:
        e = g.exponent
        if e is not None and e.symbol is not None:
            gen = tuple(sorted((tuple(sorted(t.factors.items())), t.coefficient) for t in g.generator.terms))
            out.append(("s", tuple(g.targets), symbol_index[e.symbol], e.coeff, e.const, gen))
        else:
            d = _concrete_is_diag(g)
            ax = "" if (d or g.matrix is not None) else _rotation_axis(_gate_terms(g), tuple(g.targets))
            out.append(("c", tuple(g.targets), d, CLS_GENERAL if d else _concrete_class(g), ax))
    return tuple(out)


def _class_ok(cls: int, m) -> bool:
    """Does matrix m have the structure the kernels assume for class ``cls``?"""
    if cls == CLS_GENERAL or m.shape[0] != 2:
        return True
    if cls == CLS_REAL:
        return bool(np.all(m.imag == 0))
    return bool(m[0, 0].imag == 0 and m[1, 1].imag == 0 and m[0, 1].real == 0 and m[1, 0].real == 0)


class TopologyMismatch(ValueError):
    """Rows of one bound batch differ in gate structure (ops.* then splits the batch into
    one launch sequence per topology)."""


def batch_overrides(template, circuits, symbol_index, infos) -> dict:
    """Rows of one plan must share the template's gate structure (targets, symbols,
    generators, diagonal-ness); concrete values may differ.  Returns {gate index: (cls,
    axis)} where some row's matrix does not fit the template's class / rotation axis (the
    plan then uses the general form for that gate).  Raises ValueError on structure."""
    over: dict = {}
    seen = {id(template)}
    for c in circuits:
        if id(c) in seen:
            continue
        seen.add(id(c))
        if c.num_qubits != template.num_qubits or len(c.gates) != len(template.gates):
            raise TopologyMismatch("all circuits of a batch must share one gate structure")
        for i, (gc, gt) in enumerate(zip(c.gates, template.gates)):
            if gc is gt:
                continue
            info = infos[i]
            bad = tuple(int(q) for q in gc.targets) != info.targets
            ec = gc.exponent
            sym = ec is not None and ec.symbol is not None
            if not bad and sym != info.symbolic:
                bad = True
            if not bad and sym:
                et = gt.exponent
                bad = (symbol_index.get(ec.symbol) != info.sym or ec.coeff != et.coeff or ec.const != et.const
                       or (gc.generator is not gt.generator and
                           sorted(((tuple(sorted(t.factors.items())), t.coefficient) for t in gc.generator.terms))
                           != sorted(((tuple(sorted(t.factors.items())), t.coefficient) for t in gt.generator.terms))))
            elif not bad:
                m = concrete_matrix(gc)
                if info.diag:
                    bad = not bool(np.all(m[~np.eye(m.shape[0], dtype=bool)] == 0))
                else:
                    cls, ax = over.get(i, (info.cls, info.axis))
                    if not _class_ok(cls, m):
                        cls = CLS_GENERAL
                    if ax and (gc.matrix is not None or _rotation_axis(_gate_terms(gc), info.targets) != ax):
                        ax = ""
                    if (cls, ax) != (info.cls, info.axis):
                        over[i] = (cls, ax)
            if bad:
                raise TopologyMismatch(f"gate {i} of a batch row differs in structure from the first row's "
                                 "(targets, generator, symbol, diagonal-ness); rows of one call must share "
                                 "a topology")
    return over


_DIAG_CACHE: dict = {}


def _concrete_is_diag(g) -> bool:
    if g.matrix is None:
        return _is_z_only(_gate_terms(g))
    key = id(g)
    hit = _DIAG_CACHE.get(key)
    if hit is not None and hit[0] is g:
        return hit[1]
    m = np.asarray(g.matrix)
    d = bool(np.all(m[~np.eye(m.shape[0], dtype=bool)] == 0))
    _DIAG_CACHE[key] = (g, d)
    return d


def analyse(circuit, symbol_index, overrides=None) -> list[GateInfo]:
    """``overrides``: {gate index: (cls, axis)} from batch_overrides."""
    infos = []
    for i, g in enumerate(circuit.gates):
        e = g.exponent
        tg = tuple(int(q) for q in g.targets)
        if e is not None and e.symbol is not None:
            terms = _gate_terms(g)
            infos.append(GateInfo(i, tg, True, _is_z_only(terms), symbol_index[e.symbol],
                                  float(e.coeff), float(e.const), terms, cls=_symbolic_class(terms, tg),
                                  axis=_rotation_axis(terms, tg), pstring=_pauli_string(terms, tg)))
        else:
            d = _concrete_is_diag(g)
            ax = "" if (d or g.matrix is not None) else _rotation_axis(_gate_terms(g), tg)
            cls = CLS_GENERAL if d else _concrete_class(g)
            if overrides and i in overrides:
                cls, ax = overrides[i]
            infos.append(GateInfo(i, tg, False, d, cls=cls, axis=ax))
    return infos


# ---------------------------------------------------------------------------
# ops (fusion)
# ---------------------------------------------------------------------------


@dataclass
class Op:
    kind: int
    qubits: tuple                      # DENSE: ordered (msb, lsb) / (q,); DIAG: support
    factors: list = field(default_factory=list)   # gate indices in application order (dense)
    gates: list = field(default_factory=list)     # gate indices (diag)
    symbolic: bool = False
    sym: int = -1                      # adjoint: the op's single symbol (-1 = none)
    index: int = 0
    obs: int = -1                      # OBS: observable id
    obs_terms: list = field(default_factory=list)  # OBS: [(zmask, coef column)]


def _diag_op_qubits(gates, infos):
    qs = set()
    for gi in gates:
        qs.update(infos[gi].targets)
    return tuple(sorted(qs))


FUSION_ENABLED = True   # False: one op per gate (the reference's fuse_enabled=False cells)
# forward programs: phase gates and 1q runs on a pair join the pair's dense 4x4 (QF_ABSORB_2Q=0: off)
ABSORB_INTO_2Q = __import__("os").environ.get("QF_ABSORB_2Q", "1") not in ("0", "", "false")


def build_ops(infos: list[GateInfo], adjoint: bool, block: bool = False) -> list[Op]:
    """Fuse gates into dense 1q/2q ops and diagonal phase-polynomial ops.

    ``adjoint``: symbolic gates are never merged with anything except that
    symbolic diagonal gates sharing one symbol share a DIAG op.

    ``block`` (adjoint only): symbolic gates are fused into dense blocks like in the forward
    program -- a symbolic diagonal gate joins the dense op that is the last op on all its
    qubits -- and the adjoint takes every factor's gradient from the block's reduced
    two-point matrix (see build_program / qf_block_grads).  Diagonal gates that do not land on
    a dense op keep the phase-polynomial path (QAOA cost layers stay DIAG ops).
    """
    if not FUSION_ENABLED:
        out = []
        for gi, info in enumerate(infos):
            if info.diag:
                out.append(Op(OP_DIAG, tuple(sorted(info.targets)), gates=[gi], symbolic=info.symbolic,
                              sym=info.sym if info.symbolic else -1))
            else:
                out.append(Op(OP_DENSE1 if len(info.targets) == 1 else OP_DENSE2, tuple(info.targets),
                              factors=[gi], symbolic=info.symbolic, sym=info.sym if info.symbolic else -1))
            out[-1].index = len(out) - 1
        return out
    ops: list[Op | None] = []
    last: dict[int, int] = {}   # qubit -> index of last op touching it

    def live(i):
        return ops[i] is not None

    for gi, info in enumerate(infos):
        tq = info.targets
        if info.diag and block and info.symbolic:
            js = {last.get(q) for q in tq}
            j = js.pop() if len(js) == 1 else None
            if j is not None and ops[j] is not None and ops[j].kind in (OP_DENSE1, OP_DENSE2) \
                    and set(tq) <= set(ops[j].qubits):
                ops[j].factors.append(gi)   # j is the last op on every target: exact
                ops[j].symbolic = True
                continue
        if info.diag and info.symbolic and not adjoint and ABSORB_INTO_2Q:
            # forward: a symbolic diagonal gate right after a dense two-qubit op on its qubits
            # costs nothing as a factor of that op (the 4x4 apply is paid anyway)
            js = {last.get(q) for q in tq}
            j = js.pop() if len(js) == 1 else None
            if j is not None and ops[j] is not None and ops[j].kind == OP_DENSE2 and set(tq) <= set(ops[j].qubits):
                ops[j].factors.append(gi)
                ops[j].symbolic = True
                continue
        if info.diag:
            # walk back over ops that commute with this gate (disjoint or diagonal)
            # and join the most recent compatible DIAG op
            target = None
            for j in range(len(ops) - 1, -1, -1):
                op = ops[j]
                if op is None:
                    continue
                if op.kind == OP_DIAG:
                    ok = (not adjoint) or not (info.symbolic and op.symbolic and op.sym != info.sym)
                    if ok:
                        target = j
                        break
                    continue
                if set(op.qubits) & set(tq):
                    break
            if target is not None:
                op = ops[target]
                op.gates.append(gi)
                op.qubits = _diag_op_qubits(op.gates, infos)
                if info.symbolic:
                    op.symbolic = True
                    op.sym = info.sym
                for q in tq:
                    if last.get(q, -1) < target:
                        last[q] = target
            else:
                ops.append(Op(OP_DIAG, tuple(sorted(tq)), gates=[gi], symbolic=info.symbolic,
                              sym=info.sym if info.symbolic else -1))
                for q in tq:
                    last[q] = len(ops) - 1
            continue

        can_merge_sym = (not adjoint) or block
        if len(tq) == 1:
            q = tq[0]
            j = last.get(q)
            if j is not None and ops[j] is not None and ops[j].kind in (OP_DENSE1, OP_DENSE2):
                prev = ops[j]
                if can_merge_sym or (not info.symbolic and not prev.symbolic):
                    # all later ops touching q: none (j is last on q) -> merge is exact
                    prev.factors.append(gi)
                    prev.symbolic |= info.symbolic
                    continue
            ops.append(Op(OP_DENSE1, tq, factors=[gi], symbolic=info.symbolic,
                          sym=info.sym if info.symbolic else -1))
            last[q] = len(ops) - 1
            continue

        a, b = tq
        ja, jb = last.get(a), last.get(b)
        if ja is not None and ja == jb and ops[ja].kind == OP_DENSE2 and set(ops[ja].qubits) == {a, b} \
                and (can_merge_sym or (not info.symbolic and not ops[ja].symbolic)):
            ops[ja].factors.append(gi)
            ops[ja].symbolic |= info.symbolic
            continue
        new = Op(OP_DENSE2, (a, b), factors=[], symbolic=info.symbolic,
                 sym=info.sym if info.symbolic else -1)
        if (not adjoint or block) and ABSORB_INTO_2Q:
            # forward / block-fused adjoint: every earlier op that lives on {a, b} alone and is not followed by an
            # op linking a or b to another qubit joins the new 4x4 (1q runs, symbolic phase
            # gates on a / b / the pair): later ops touching them are absorbed too, ops on
            # other qubits commute with them
            pair, blocked, take = {a, b}, set(), []
            for j in range(len(ops) - 1, -1, -1):
                op = ops[j]
                if op is None or not (set(op.qubits) & pair):
                    continue
                qs = set(op.qubits)
                ok = qs <= pair and not (qs & blocked) and (
                    op.kind == OP_DENSE1 or (op.kind == OP_DIAG and all(infos[g].symbolic for g in op.gates)))
                if ok:
                    take.append(j)
                else:
                    blocked |= qs & pair
                    if blocked == pair:
                        break
            for j in reversed(take):
                new.factors.extend(ops[j].factors if ops[j].kind == OP_DENSE1 else ops[j].gates)
                new.symbolic |= ops[j].symbolic
                ops[j] = None
        # absorb trailing 1q dense ops on a / b (they are the last op on their qubit)
        for q in (a, b):
            j = last.get(q)
            if j is not None and ops[j] is not None and ops[j].kind == OP_DENSE1 and \
                    (can_merge_sym or (not info.symbolic and not ops[j].symbolic)):
                new.factors.extend(ops[j].factors)
                new.symbolic |= ops[j].symbolic
                ops[j] = None
        new.factors.append(gi)
        ops.append(new)
        last[a] = last[b] = len(ops) - 1

    out = [o for o in ops if o is not None]
    if block:
        out = _split_small_blocks(out, infos)
    for i, o in enumerate(out):
        o.index = i
    return out


BLOCK_MIN_SYMBOLIC = 3


def _split_small_blocks(ops: list, infos) -> list:
    """Keep a fused symbolic block only where it pays: a two-qubit block with at least
    BLOCK_MIN_SYMBOLIC symbolic factors (one dense 4x4 apply and a 16-entry A matrix instead
    of a per-gate sweep).  Smaller blocks -- and every one-qubit run, whose per-gate
    normalised rotations are as cheap and keep the Pauli frame and the checkpointed adjoint
    available -- go back to one op per gate, in place (exact: a merged gate was the last op
    on its qubits)."""
    res = []
    for o in ops:
        nsym = sum(infos[gi].symbolic for gi in o.factors)
        if o.kind in (OP_DENSE1, OP_DENSE2) and o.symbolic and len(o.factors) > 1 and \
                not (o.kind == OP_DENSE2 and nsym >= BLOCK_MIN_SYMBOLIC):
            for gi in o.factors:
                inf = infos[gi]
                sym = inf.sym if inf.symbolic else -1
                if inf.diag:
                    res.append(Op(OP_DIAG, tuple(sorted(inf.targets)), gates=[gi], symbolic=inf.symbolic, sym=sym))
                else:
                    res.append(Op(OP_DENSE1 if len(inf.targets) == 1 else OP_DENSE2, tuple(inf.targets),
                                  factors=[gi], symbolic=inf.symbolic, sym=sym))
        else:
            res.append(o)
    return res


def dependencies(ops: list[Op]) -> list[set]:
    """preds[j]: ops that must run before j (diagonal ops commute with each other)."""
    last_nd: dict[int, int] = {}
    diag_since: dict[int, list] = {}
    preds = []
    for j, op in enumerate(ops):
        p = set()
        is_diag = op.kind in (OP_DIAG, OP_OBS)
        for q in op.qubits:
            if q in last_nd:
                p.add(last_nd[q])
            if not is_diag:
                p.update(diag_since.get(q, []))
        preds.append(p)
        for q in op.qubits:
            if is_diag:
                diag_since.setdefault(q, []).append(j)
            else:
                last_nd[q] = j
                diag_since[q] = []
    return preds


def absorb_product_init(ops: list[Op], infos, n: int, allow_symbolic: bool):
    """Leading 1q dense ops become the product-state initialisation."""
    first: dict[int, int] = {}
    for j, op in enumerate(ops):
        for q in op.qubits:
            first.setdefault(q, j)
    init = {}
    keep = []
    for j, op in enumerate(ops):
        if op.kind == OP_DENSE1 and first.get(op.qubits[0]) == j and (allow_symbolic or not op.symbolic):
            init[op.qubits[0]] = op
        else:
            keep.append(op)
    for i, o in enumerate(keep):
        o.index = i
    return keep, init


# ---------------------------------------------------------------------------
# passes and stages
# ---------------------------------------------------------------------------


@dataclass
class Stage:
    regs: list            # local bits in register slots (slot j -> regs[j])
    ops: list             # Op objects in execution order
    lane: set = field(default_factory=set)   # ids of ops applied on a lane bit (warp shuffles)


@dataclass
class Pass:
    qubits: list          # logical qubits of the tile, local bit i -> qubits[i] (ascending physical position)
    ops: list
    stages: list = field(default_factory=list)
    init: int = INIT_LOAD
    store: int = 1
    # qubit relabelling (plan_passes_remap): physical position of every logical qubit when the
    # pass loads (None: identity), and the physical position local bit i is stored to
    pos_in: list = None
    out_pos: list = None


class _Sched:
    def __init__(self, ops, subset=None):
        self.ops = ops
        ids = set(range(len(ops))) if subset is None else set(subset)
        preds = dependencies(ops)
        self.npred = {j: len([p for p in preds[j] if p in ids]) for j in ids}
        self.succ = {j: [] for j in ids}
        for j in ids:
            for p in preds[j]:
                if p in ids:
                    self.succ[p].append(j)
        self.ready = [j for j in ids if self.npred[j] == 0]
        heapq.heapify(self.ready)
        self.left = len(ids)

    def take(self, j):
        self.left -= 1
        for s in self.succ[j]:
            self.npred[s] -= 1
            if self.npred[s] == 0:
                heapq.heappush(self.ready, s)

    def drain(self, fits):
        """Repeatedly take ready ops accepted by ``fits``; return them in order."""
        taken = []
        while True:
            pick = None
            for j in sorted(self.ready):
                if fits(self.ops[j]):
                    pick = j
                    break
            if pick is None:
                return taken
            self.ready.remove(pick)
            heapq.heapify(self.ready)
            self.take(pick)
            taken.append(self.ops[pick])


def plan_passes(ops: list[Op], n: int, L: int) -> list[Pass]:
    if n == L:
        return [Pass(list(range(n)), list(ops))] if ops else [Pass(list(range(n)), [])]
    sch = _Sched(ops)
    passes = []
    while sch.left > 0:
        Q = set(range(LANE_Q))
        taken = []
        while True:
            taken += sch.drain(lambda o: o.kind in (OP_DIAG, OP_OBS) or set(o.qubits) <= Q)
            cands = [sch.ops[j] for j in sch.ready]
            if not cands:
                break
            best = min(cands, key=lambda o: (len(set(o.qubits) - Q), o.index))
            if len(Q | set(best.qubits)) > L:
                break
            Q |= set(best.qubits)
        if not taken:
            raise AssertionError("pass planner made no progress")
        for q in range(n):
            if len(Q) >= L:
                break
            Q.add(q)
        passes.append(Pass(sorted(Q), taken))
    if not passes:
        passes.append(Pass(list(range(L)), []))
    return passes


def _sched_copy(sch: "_Sched") -> "_Sched":
    c = object.__new__(_Sched)
    c.ops, c.succ = sch.ops, sch.succ
    c.npred = dict(sch.npred)
    c.ready = list(sch.ready)
    c.left = sch.left
    return c


def _greedy_tile(sch: "_Sched", Q: set, L: int) -> list:
    """The plan_passes greedy on ``sch`` (mutated) from tile ``Q`` (mutated): ops taken."""
    taken = []
    while True:
        taken += sch.drain(lambda o: o.kind in (OP_DIAG, OP_OBS) or set(o.qubits) <= Q)
        cands = [sch.ops[j] for j in sch.ready]
        if not cands:
            break
        best = min(cands, key=lambda o: (len(set(o.qubits) - Q), o.index))
        if len(Q | set(best.qubits)) > L:
            break
        Q |= set(best.qubits)
    return taken


def _wanted(sch: "_Sched", L: int) -> list:
    """Qubits the next pass would choose with no lane constraint, in the order it adds them."""
    c = _sched_copy(sch)
    Q: set = set()
    order = []
    while True:
        c.drain(lambda o: o.kind in (OP_DIAG, OP_OBS) or set(o.qubits) <= Q)
        cands = [c.ops[j] for j in c.ready]
        if not cands:
            break
        best = min(cands, key=lambda o: (len(set(o.qubits) - Q), o.index))
        if len(Q | set(best.qubits)) > L:
            break
        for q in best.qubits:
            if q not in Q:
                order.append(q)
        Q |= set(best.qubits)
    return order


def plan_passes_remap(ops: list[Op], n: int, L: int) -> list[Pass]:
    """plan_passes with qubit relabelling.  Physical bits 0..3 must be tile bits of every pass
    (lanes 0-15 move 128 contiguous bytes), which in plan_passes wastes 4 of the L tile qubits
    whenever the pending gates sit on high qubits (brickwork circuits: passes of 6 gates).  Here
    each pass stores its tile back with a permutation of the tile's physical positions: the
    qubits the NEXT pass wants (its greedy choice without the lane constraint) are moved onto
    physical bits 0..3.  Every pass records the layout it loads (pos_in) and the position each
    local bit is stored to (out_pos); the program's final layout is in Program.final_pos.
    cfg5 (32 qubits, depth 14, L = 11): 26 -> 15 passes."""
    if n == L:
        return plan_passes(ops, n, L)
    sch = _Sched(ops)
    pos = list(range(n))          # logical -> physical
    at = list(range(n))           # physical -> logical
    passes = []
    while sch.left > 0:
        Q = {at[p] for p in range(LANE_Q)}
        taken = _greedy_tile(sch, Q, L)
        if not taken:
            raise AssertionError("pass planner made no progress")
        want = _wanted(sch, L)
        for q in want + sorted(range(n), key=lambda q: pos[q]):
            if len(Q) >= L:
                break
            Q.add(q)
        P = sorted(pos[q] for q in Q)
        qubits = [at[p] for p in P]
        nxt = [q for q in want if q in Q][:LANE_Q]
        order = nxt + [q for q in qubits if q not in nxt]
        new_pos = {q: P[i] for i, q in enumerate(order)}
        out_pos = [new_pos[q] for q in qubits]
        passes.append(Pass(qubits, taken, pos_in=list(pos), out_pos=out_pos))
        for q, p_ in new_pos.items():
            pos[q] = p_
            at[p_] = q
    return passes


def _stage_regs(need: set, R: int, L: int, lanes: set, prefer: list) -> list:
    regs = set(need)
    for b in prefer + list(range(L - 1, -1, -1)):
        if len(regs) >= R:
            break
        if b in regs or b in lanes:
            continue
        regs.add(b)
    return sorted(regs)


def plan_stages(p: Pass, R: int, vec: bool = False, lane_ok=None) -> None:
    """Register stages of one tile pass.  ``vec``: 16-byte edge accesses -- the first and
    (where its registers allow) the last stage hold local bit 0 = qubit 0 in register slot 0
    and take local bits 1..LANE_Q as lanes, so a thread loads / stores amplitude pairs
    (x, x | 1) as one float4 (LDG.128 / STG.128, 256-byte runs per 16 lanes)."""
    L = len(p.qubits)
    loc = {q: i for i, q in enumerate(p.qubits)}
    ops = p.ops
    sch = _Sched(ops)
    stages: list[Stage] = []
    # only where local bits 0..LANE_Q are qubits 0..LANE_Q (runs of >= 256 bytes): on tiles with
    # 128-byte runs the pair layout spreads a warp over twice as many runs and measured slower
    # (headline forward passes 1/3: 0.748 -> 0.830 ms; contiguous pass 2: 0.802 -> 0.796 ms,
    # backward pass 2: 2.118 -> 2.067 ms)
    vec = vec and p.out_pos is None and list(p.qubits[:LANE_Q + 1]) == list(range(LANE_Q + 1)) and L - R > LANE_Q
    edge_lanes = set(range(1, LANE_Q + 1)) if vec else set(range(LANE_Q))

    def local_set(o):
        return {loc[q] for q in o.qubits}

    while sch.left > 0:
        first = not stages
        # choose register bits: greedily cover ready dense ops (in index order)
        need: set = {0} if (first and vec) else set()
        virt = _Sched(ops, subset=[j for j in range(len(ops)) if j in sch.npred and sch.npred.get(j, 0) >= 0])
        # replay the real state into the virtual scheduler
        virt.npred = dict(sch.npred)
        virt.ready = list(sch.ready)
        heapq.heapify(virt.ready)
        virt.left = sch.left
        while True:
            progressed = False
            for j in sorted(virt.ready):
                o = ops[j]
                if o.kind in (OP_DIAG, OP_OBS):
                    virt.ready.remove(j); heapq.heapify(virt.ready); virt.take(j)
                    progressed = True
                    break
                ls = local_set(o)
                if first and ls & edge_lanes:
                    continue
                if len(need | ls) <= R:
                    need |= ls
                    virt.ready.remove(j); heapq.heapify(virt.ready); virt.take(j)
                    progressed = True
                    break
            if not progressed:
                break
        upcoming = []
        for j in sorted(virt.ready):
            for b in sorted(local_set(ops[j])):
                if b not in upcoming:
                    upcoming.append(b)
        regs = _stage_regs(need, R, L, lanes=edge_lanes if first else set(),
                           prefer=[b for b in upcoming if b not in edge_lanes])
        rs = set(regs)
        taken = sch.drain(lambda o: o.kind in (OP_DIAG, OP_OBS) or local_set(o) <= rs)
        stages.append(Stage(regs, taken))
        if not taken and not first:
            raise AssertionError("stage planner made no progress")
    if not stages:
        stages.append(Stage(sorted({0} | set(range(L - R + 1, L))) if vec else list(range(L - R, L)), []))
    if lane_ok is not None and LANE_OPS > 0 and p.out_pos is None and len(stages) >= 2:
        # lane ops: merge the last two stages into one edge-layout stage when the gates that do
        # not fit its registers are normalised X rotations on its first LANE_Q lane bits (the
        # edge lanes), applied with warp shuffles -- one shared-memory exchange fewer
        a_, b_ = stages[-2], stages[-1]
        merged = list(a_.ops) + list(b_.ops)
        need_r = {0} if vec else set()
        lane_ops = []
        for o in merged:
            if o.kind in (OP_DIAG, OP_OBS):
                continue
            ls = local_set(o)
            if len(ls) == 1 and ls <= edge_lanes and lane_ok(o):
                lane_ops.append(o)
            else:
                need_r |= ls
        if lane_ops and len(lane_ops) <= LANE_OPS and not need_r & edge_lanes and len(need_r) <= R:
            regs = _stage_regs(need_r, R, L, lanes=edge_lanes,
                               prefer=[b for b in b_.regs + a_.regs if b not in edge_lanes])
            stages[-2:] = [Stage(regs, merged, {id(o) for o in lane_ops})]
            p.stages = stages
            return
    if vec:
        # 16-byte stores from the last stage when its ops leave local bit 0 a register slot
        # and keep off the lanes 1..LANE_Q (else the 8-byte store rule below)
        last = stages[-1]
        used = set()
        for o in last.ops:
            if o.kind not in (OP_DIAG, OP_OBS):
                used |= local_set(o)
        if not used & edge_lanes and (0 in used or len(used) < R):
            last.regs = _stage_regs(used | {0}, R, L, lanes=edge_lanes,
                                    prefer=[b for b in last.regs if b not in edge_lanes])
            p.stages = stages
            return
    # the store needs lanes on the local bits stored to physical 0..3: local 0..3, or for a
    # relabelled pass the bits whose out_pos < 4 (then the load and store stages differ)
    sl = store_lanes(p)
    if set(stages[-1].regs) & set(sl) or (len(stages) == 1 and sl != list(range(LANE_Q))):
        free = [b for b in range(L - 1, -1, -1) if b not in sl]
        stages.append(Stage(sorted(free[:R]), []))
    p.stages = stages


def store_lanes(p: Pass) -> list:
    """Local bits the pass stores to physical bits 0..LANE_Q-1, in that order."""
    if p.out_pos is None:
        return list(range(LANE_Q))
    return [p.out_pos.index(k) for k in range(LANE_Q)]


def stage_slots(p: Pass, st: Stage, R: int, edge: bool = True, lanes: list = None):
    """(register local bits, thread local bits [lanes first]).

    Edge stages (a pass's first / last, which load / store global memory) keep the lowest
    free bits as lanes (local bits 0..3: 128-byte runs).  Inner stages only exchange through
    shared memory, whose 64-bit accesses are conflict-free when the 16 lanes of a half-warp
    hit 16 distinct 8-byte bank pairs: with ``swizzle`` the low nibble of local bit b is bit
    b mod 4, so lanes 0..3 take free bits of four distinct classes mod 4 where possible."""
    L = len(p.qubits)
    rs = set(st.regs)
    free = [b for b in range(L) if b not in rs]
    if lanes is not None:     # a relabelled pass's store stage: its store lanes first
        return list(st.regs), list(lanes) + [b for b in free if b not in lanes]
    if edge or CONFLICT_FREE_LANES is False:
        return list(st.regs), free
    lanes, seen = [], set()
    for b in free:
        if len(lanes) < LANE_Q and b % 4 not in seen:
            lanes.append(b)
            seen.add(b % 4)
    if len(lanes) < LANE_Q:
        return list(st.regs), free
    return list(st.regs), lanes + [b for b in free if b not in lanes]


CONFLICT_FREE_LANES = __import__("os").environ.get("QF_LANE_ORDER", "1") not in ("0", "", "false")
# qubit relabelling between passes (plan_passes_remap): plan-specialised forward programs without
# Pauli frames / checkpoints / caller states.  Measured: cfg5 26 -> 16 passes but 620 -> 601 ms,
# cfg4 22 -> 14 passes but 162 -> 186 ms -- dense brickwork passes are FMA-bound (217 fused
# blocks x 8 FFMA2 per amplitude = 0.40 s floor at 32 qubits), so fewer HBM passes buy little
# and the extra store stages cost more; off by default
# lane ops (plan_stages ``lane_ok``): at most this many warp-shuffle rotations in a pass's
# merged last stage (0: off).  Measured on the headline (one B200): one register stage and one
# shared-memory exchange fewer per pass, but forward passes 0.746 -> 0.850 ms and backward
# passes 2.06 -> 2.23 ms -- a lane rotation moves every amplitude's partner through SHFL (8 B
# per amplitude and state), the exchange it replaces serves 4-9 gates; off by default
LANE_OPS = int(__import__("os").environ.get("QF_LANE_OPS", "0"))
# 16-byte edge loads / stores in plan-specialised kernels (plan_stages ``vec``)
VEC_EDGE = __import__("os").environ.get("QF_VEC_EDGE", "1") not in ("0", "", "false")
REMAP = __import__("os").environ.get("QF_REMAP", "0") not in ("0", "", "false")
# tensor-core stages (csrc/qf_tc.cu): forward dense programs at 16 x 128 amplitudes per tile;
# a stage qualifies when its dense work is at least TC_MIN_FFMA2 FFMA2 per amplitude.
# Measured (one B200): cfg4 161 -> 172 ms, cfg5 614 -> 688 ms (per-stage B staging, barriers and
# MMA round trips outweigh the FFMA2 work of 2-3 fused blocks), and the tensor cores' fp32
# accumulation shrinks every block's output by ~1.4e-6 (24q depth 20: norm 1 - 1.1e-4) -- off
# by default
TC_STAGES = __import__("os").environ.get("QF_TC", "0") not in ("0", "", "false")
TC_MIN_FFMA2 = int(__import__("os").environ.get("QF_TC_MIN", "16"))


# ---------------------------------------------------------------------------
# program emission
# ---------------------------------------------------------------------------


@dataclass
class Program:
    n: int
    L: int
    R: int
    adjoint: bool
    passes: np.ndarray            # [P, 128] int32
    stages: np.ndarray            # [S, 64] int32
    ops: np.ndarray               # [O, 16] int32
    term_mask: np.ndarray         # uint32
    term_idx: np.ndarray          # int32
    term_w: np.ndarray            # float32
    grp: np.ndarray               # int32
    genmats: np.ndarray           # float32 interleaved complex
    n_slots: int
    n_mat: int
    n_ang: int
    n_coef: int
    # build recipe
    recipe: dict
    # slot -> output mapping
    grad_slots: dict              # symbol column -> [slots]
    obs_slots: dict               # observable id -> [slots]
    energy_slots: list
    stats: dict
    frame: bool = False
    frame_events: np.ndarray = None   # [E, EV_INTS] int32, execution order
    # block-fused adjoint (build_ops(block=True)): per block [factor begin, factor end, D,
    # first A slot]; per factor [mat offset, generator offset (-1: fixed), symbol column];
    # block_gens: complex D x D generators 2 coeff G (non-identity part), interleaved float64
    blocks: np.ndarray = None
    block_factors: np.ndarray = None
    block_gens: np.ndarray = None
    # qubit relabelling (plan_passes_remap): physical bit of every logical qubit after the last
    # pass (None: identity layout)
    final_pos: list = None
    # tensor-core stages: per block [(op kind, matrix offset, slot 0, slot 1)] in application
    # order; stage row [50] = block index + 1
    tc_blocks: list = None


def _bit_subset(mask: int, reg_glob: list) -> int:
    s = 0
    for j, g in enumerate(reg_glob):
        if mask >> g & 1:
            s |= 1 << j
    return s


class Emitter:
    def __init__(self, n, L, R, infos, adjoint):
        self.n, self.L, self.R, self.infos, self.adjoint = n, L, R, infos, adjoint
        self.pass_rows, self.stage_rows, self.op_rows = [], [], []
        self.term_mask, self.term_idx, self.term_w, self.grp = [], [], [], []
        self.genmats = []
        self.n_mat = 0
        self.n_ang = 0
        self.n_coef = 0
        self.n_slots = 0
        self.dense_recipe = []    # (mat offset, dim, factors[(kind, src, emb)])
        self.term_src = []        # (kind, src, beta)
        self.grad_slots: dict = {}
        self.obs_slots: dict = {}
        self.energy_slots: list = []
        self.coef_cols = []       # (obs id, term index within observable)
        self.blocks = []          # (factor gate indices, order, D, first A slot)
        self.tc_blocks = []       # tensor-core stages: [(op kind, matrix offset, slot 0, slot 1)]

    # -- per-row matrix slab --------------------------------------------------
    def dense_mat(self, op: Op, order: tuple) -> int:
        """Reserve slab space for a dense op whose local basis is ``order`` (msb first)."""
        d = 1 << len(order)
        off = self.n_mat
        self.n_mat += d * d
        facs = []
        for gi in op.factors:
            info = self.infos[gi]
            kind, src = (0, info.gen) if info.symbolic else (1, info.fixed)
            if len(order) == 1:
                emb = 4
            elif len(info.targets) == 2:
                emb = 0 if tuple(info.targets) == tuple(order) else 1
            else:
                emb = 2 if info.targets[0] == order[0] else 3
            facs.append((kind, src, emb))
        self.dense_recipe.append((off, d, facs))
        return off

    def angle_col(self, kind, src, beta) -> int:
        self.term_src.append((kind, src, beta))
        self.n_ang += 1
        return self.n_ang - 1

    def emit_terms(self, terms, reg_glob):
        """terms: [(zmask, idx, weight)] -> sorted by register subset; returns (begin, end, grp)."""
        R = self.R
        keyed = sorted(((_bit_subset(m, reg_glob), m, i, w) for m, i, w in terms), key=lambda x: x[0])
        begin = len(self.term_mask)
        bounds = [begin] * ((1 << R) + 1)
        for s, m, i, w in keyed:
            self.term_mask.append(m)
            self.term_idx.append(i)
            self.term_w.append(w)
        pos = begin
        k = 0
        for S in range(1 << R):
            bounds[S] = pos
            while k < len(keyed) and keyed[k][0] == S:
                k += 1
                pos += 1
        bounds[1 << R] = pos
        g = len(self.grp)
        self.grp.extend(bounds)
        return begin, len(self.term_mask), g

    def diag_terms(self, op: Op):
        """Phase-polynomial terms of a DIAG op: [(zmask, angle column, grad weight)]."""
        out = []
        for gi in op.gates:
            info = self.infos[gi]
            if info.symbolic:
                for f, beta in info.terms:
                    zm = 0
                    for q in f:
                        zm |= 1 << q
                    col = self.angle_col(0, info.gen, beta)
                    w = 2.0 * info.coeff * beta if (self.adjoint and zm) else 0.0
                    out.append((zm, col, w))
            else:
                k = len(info.targets)
                for s in range(1 << k):
                    zm = 0
                    for j in range(k):  # walsh index bit j <-> targets[k-1-j] (msb = targets[0])
                        if s >> j & 1:
                            zm |= 1 << info.targets[k - 1 - j]
                    col = self.angle_col(1, info.const_col + s, 0.0)
                    out.append((zm, col, 0.0))
        return out

    def new_slot(self) -> int:
        self.n_slots += 1
        return self.n_slots - 1


def _walsh_angles(diag_entries: np.ndarray) -> np.ndarray:
    """Angles a_s (s over subsets of local bits, bit j <-> local bit j from the LSB) with
    diag[x] = exp(-i sum_s a_s (-1)^{popc(s & x)})."""
    phi = -np.angle(diag_entries)
    d = phi.shape[-1]
    a = phi.copy()
    h = 1
    while h < d:
        for i in range(0, d, 2 * h):
            x = a[..., i:i + h].copy()
            y = a[..., i + h:i + 2 * h].copy()
            a[..., i:i + h] = x + y
            a[..., i + h:i + 2 * h] = x - y
        h *= 2
    return a / d


def has_normalisable(ops: list[Op], infos) -> bool:
    """Does any op become a Pauli-frame normalised rotation?  Without one the frame stays the
    identity (dense ops absorb it, diagonal ops see no x part) and the walk is wasted work."""
    for o in ops:
        if o.kind == OP_DENSE1:
            axes = {infos[gi].axis for gi in o.factors}
            if len(axes) == 1 and axes <= {"X", "Y"}:
                return True
        elif (o.kind == OP_DENSE2 and len(o.factors) == 1 and infos[o.factors[0]].symbolic
              and bool(infos[o.factors[0]].pstring)):
            return True
    return False


def frame_eligible(ops: list[Op], infos, adjoint: bool) -> bool:
    """Every program qualifies: normalised X/Y rotations carry their generator's frame sign
    in the slot scale; any other gradient-carrying dense op absorbs the frame into its matrix
    and evaluates its gradient after applying U^dag (G commutes with U), where the frame on
    its qubits is the identity."""
    return True


def block_slots(D: int) -> int:
    """A slots of a D x D block: D diagonal entries + Re/Im of the D(D-1)/2 upper ones."""
    return D * D


def build_program(circuit_template, infos: list[GateInfo], n: int, adjoint: bool,
                  observables=None, obs_diag_ids=(), lam_diag: bool = False,
                  from_state: bool = False, frame: bool = False, mirror: bool = False,
                  block: bool = False, jit: bool = False, vec: bool = None) -> Program:
    """Plan + emit.  ``observables``: list of PauliSums; ``obs_diag_ids``: those fused as
    OBS ops at the end of the forward program; ``lam_diag``: adjoint with a diagonal H
    whose lambda-init / energy is fused into the first backward pass; ``from_state``:
    the forward program starts from a caller-provided state instead of |0...0>.

    ``frame``: Pauli-frame normalisation (see csrc/qf_capi.cu frame_walk_kernel).  Single-
    qubit X/Y rotations c I - i s P are applied as I - i tau P (|tau| <= 1, one FFMA2 per
    amplitude); the stored state is psi = sqrt(m) X^x Z^z psi_stored up to a global phase,
    and the per-row frame (x, z, m) is tracked by the build step in execution order:
    general dense ops absorb the frame into their matrix, diagonal ops / observables are
    evaluated at index ^ x, and slot sums are scaled by m (and the generator's sign).

    ``vec``: the program runs as plan-specialised kernels (16-byte edge accesses,
    plan_stages); default ``jit``."""
    vec = jit if vec is None else vec
    # mirror: a forward program with exactly the adjoint program's ops and tile passes (no
    # symbolic fusion, adjoint tile size), so its pass outputs are checkpoints the adjoint
    # sweep can read and both Pauli-frame walks agree at every pass boundary
    # a mirror program takes the block-mode op list too (same ops per pass as the adjoint)
    block = block and (adjoint or mirror)
    ops = build_ops(infos, adjoint or mirror, block=block)
    L, R = geometry(adjoint)
    if adjoint and jit and "QF_GEOM_ADJ" not in __import__("os").environ and \
            all(o.kind in (OP_DENSE1, OP_DIAG, OP_OBS) for o in ops):
        # rotation / phase-polynomial programs (QAOA, HEA): 32 amplitudes of psi and lambda
        # per thread, 2 CTAs x 4 warps per SM -- fewer stage exchanges per gate; measured
        # on the headline's middle backward passes 2.20 -> 2.13 ms (R = 4: 16 warps per SM).
        # Plan-specialised kernels only (``jit``): the interpreted kernel has R = 4 adjoints
        L, R = ADJ_L, 5
    if mirror:
        L = geometry(True)[0]
    elif not adjoint and R == 5 and "QF_GEOM_FWD" not in __import__("os").environ:
        # dense two-qubit blocks hold 16 matrix pairs in registers: with 32 amplitudes per
        # thread they spill, so programs with many of them use 16 amplitudes per thread
        n2 = sum(o.kind == OP_DENSE2 for o in ops)
        if n2 * 2 > len(ops):
            L, R = 11, 4   # FP32-bound dense programs: smaller tiles, more CTAs (RCS 24q: 162 vs 167 ms)
    L = min(L, n)
    if L - R < 6 and "QF_GEOM_ADJ" not in __import__("os").environ and "QF_GEOM_FWD" not in __import__("os").environ:
        # registers that cover the whole state: at least two warps per tile (cfg1 parameter-shift
        # batches, 10 qubits: R = 4 12.7 ms vs R = 5 15.5 ms, R = 3 13.6 ms)
        R = max(4, L - 6)
    frame = frame and frame_eligible(ops, infos, adjoint)
    if from_state and not adjoint:
        init = {}
    else:
        ops, init = absorb_product_init(ops, infos, n, allow_symbolic=not (adjoint or mirror))
    # observable ops
    obs_ops = []
    if not adjoint:
        for oid in obs_diag_ids:
            obs_ops.append(Op(OP_OBS, tuple(range(n)), obs=oid))
    if frame and REMAP and jit and not adjoint and not mirror and not from_state and n > L:
        # a Pauli frame only pays off through normalised rotations; a program whose dense ops
        # would all absorb it (brickwork / RCS) is relabelled instead
        if not has_normalisable(ops, infos):
            frame = False
    remap = (REMAP and jit and not adjoint and not mirror and not from_state and not frame and n > L)
    tc_ok = TC_STAGES and jit and not adjoint and not mirror and R == 4 and L - R == 7
    passes = plan_passes_remap(ops, n, L) if remap else plan_passes(ops, n, L)
    if remap and all(p.out_pos == [p.pos_in[q] for q in p.qubits] for p in passes):
        remap = False                          # nothing moved: the plain layout
        for p in passes:
            p.pos_in = p.out_pos = None
    final_pos = list(range(n))
    if remap:
        final_pos = list(passes[-1].pos_in)
        for q, o in zip(passes[-1].qubits, passes[-1].out_pos):
            final_pos[q] = o
    def lane_ok(op):
        """Ops the plan-specialised kernels can apply on a lane bit: Pauli-frame normalised X
        rotations (class CLS_NX) with, in the adjoint, a single-X generator gradient."""
        if not (frame and op.kind == OP_DENSE1) or {infos[gi].axis for gi in op.factors} != {"X"}:
            return False
        if adjoint and op.symbolic:
            return len(op.factors) == 1 and _generator_kind(infos[op.factors[0]].terms) == GK_X
        return True

    for p in passes:
        plan_stages(p, R, vec=VEC_EDGE and vec, lane_ok=lane_ok if (vec and LANE_OPS > 0) else None)
    if obs_ops:
        passes[-1].stages[-1].ops.extend(obs_ops)
    if adjoint and lam_diag:
        obs_ops = [Op(OP_OBS, tuple(range(n)), obs=0)]

    em = Emitter(n, L, R, infos, adjoint)
    events = []
    # -- generator / fixed tables for the build recipe
    gen_rows = []
    n_fixed = 0
    n_const = 0
    for info in infos:
        if info.symbolic:
            info.gen = len(gen_rows)
            gen_rows.append(info)
        elif info.diag:
            info.const_col = n_const
            n_const += 1 << len(info.targets)
        else:
            info.fixed = n_fixed
            n_fixed += 1

    seq = list(passes)
    if adjoint:
        seq = list(reversed(passes))
    for pi, p in enumerate(seq):
        first_fwd = p is passes[0]
        last_fwd = p is passes[-1]
        stages = list(reversed(p.stages)) if adjoint else list(p.stages)
        prow = np.zeros(PASS_INTS, dtype=np.int32)
        prow[0] = len(em.stage_rows)
        if adjoint:
            prow[2] = (INIT_LOAD_PSI if lam_diag else INIT_LOAD) if last_fwd else INIT_LOAD
            prow[3] = 0 if first_fwd else 1
        else:
            prow[2] = INIT_LOAD if (from_state or not first_fwd) else (INIT_PRODUCT if init else INIT_ZERO)
            prow[3] = 1
        prow[4] = em.n_mat
        prow[6] = em.n_ang
        prow[8] = em.n_slots
        prow[11] = em.n_coef
        prow[13] = L
        prow[14] = len(em.term_mask)
        prow[80] = len(em.grp)
        prow[82] = len(em.op_rows)
        posi = p.pos_in if p.pos_in is not None else list(range(n))   # logical -> physical at load

        def phys_mask(m, posi=posi):
            out = 0
            for q in range(n):
                if m >> q & 1:
                    out |= 1 << posi[q]
            return out

        outer = sorted(posi[q] for q in range(n) if q not in set(p.qubits))
        prow[10] = len(outer)
        prow[16:16 + len(outer)] = outer
        if p.out_pos is not None:
            prow[84:84 + len(p.out_pos)] = p.out_pos
            prow[126] = 1
        prow[48:80] = -1
        if not adjoint and first_fwd:
            for q, op in sorted(init.items()):
                prow[48 + q] = em.dense_mat(op, (q,))
        fwd_index = passes.index(p)
        if frame and adjoint:
            events.append([EV_PASS, -1, -1, -1, -1, -1, fwd_index, 0])
        # slot merging (adjoint, frame-normalised X/Y rotations): rotations of one pass that
        # share a symbol and a generator weight accumulate into ONE gradient slot in registers;
        # each carries its per-row frame scale relative to the group head (written by the
        # frame walk next to tau), so the slot needs one store and one reduction per tile
        merge_heads: dict = {}
        for si, st in enumerate(stages):
            regs, thr = stage_slots(p, st, R, edge=st is p.stages[0] or st is p.stages[-1],
                                    lanes=store_lanes(p) if (p.out_pos is not None and st is p.stages[-1]) else None)
            srow = np.zeros(STAGE_INTS, dtype=np.int32)
            reg_log = [p.qubits[b] for b in regs]
            reg_glob = [posi[q] for q in reg_log]          # physical positions
            srow[0:R] = reg_glob
            srow[8:8 + len(thr)] = [posi[p.qubits[b]] for b in thr]
            srow[24:24 + R] = [swizzle(1 << b) for b in regs]
            srow[32:32 + len(thr)] = [swizzle(1 << b) for b in thr]
            srow[48] = len(em.op_rows)
            slot_of = {q: j for j, q in enumerate(reg_log)}
            st_ops = list(reversed(st.ops)) if adjoint else list(st.ops)
            if adjoint and lam_diag and last_fwd and si == 0:
                st_ops = obs_ops + st_ops
            for op in st_ops:
                orow = np.full(OP_INTS, 0, dtype=np.int32)
                orow[0] = op.kind
                orow[7] = -1
                orow[8] = -1
                orow[11] = -1
                if op.kind in (OP_DENSE1, OP_DENSE2):
                    if op.kind == OP_DENSE1 and id(op) in st.lane:
                        # lane op: thread bit (orow[15] - 1) of this stage's layout, no register slot
                        order = (op.qubits[0],)
                        orow[1] = -1
                        orow[15] = 1 + thr.index(p.qubits.index(op.qubits[0]))
                        assert orow[15] <= 5
                    elif op.kind == OP_DENSE1:
                        order = (op.qubits[0],)
                        orow[1] = slot_of[op.qubits[0]]
                    else:
                        a, b = op.qubits
                        order = (a, b) if slot_of[a] < slot_of[b] else (b, a)
                        orow[1], orow[2] = slot_of[order[0]], slot_of[order[1]]
                    orow[3] = em.dense_mat(op, order)
                    is_block = adjoint and op.symbolic and len(op.factors) > 1
                    if op.kind == OP_DENSE1:
                        cl = {infos[gi].cls for gi in op.factors}
                        orow[9] = cl.pop() if len(cl) == 1 else CLS_GENERAL
                        axes = {infos[gi].axis for gi in op.factors}
                        if frame and len(axes) == 1 and axes <= {"X", "Y"}:
                            orow[9] = CLS_NX if axes == {"X"} else CLS_NY
                        elif frame and orow[9] == CLS_XLIKE:
                            orow[9] = CLS_GENERAL   # an absorbed X frame breaks the X-like structure
                                                    # (real matrices stay real under X^a Z^b)
                        if is_block:
                            orow[9] = CLS_GENERAL   # the A matrix is taken frame-free after U^dag
                    else:
                        orow[9] = CLS_GENERAL
                        if frame and len(op.factors) == 1 and infos[op.factors[0]].symbolic and \
                                infos[op.factors[0]].pstring and not is_block:
                            orow[9] = CLS_NP
                    ev = None
                    if frame:
                        if op.kind == OP_DENSE1:
                            kind = {CLS_NX: EV_NX, CLS_NY: EV_NY}.get(int(orow[9]), EV_ABS1)
                            ev = [kind, order[0], -1, int(orow[3]), -1, -1, 0, 0]
                        elif orow[9] == CLS_NP:
                            ps = dict(infos[op.factors[0]].pstring)
                            code = PAULI_CODE[ps[order[0]]] | (PAULI_CODE[ps[order[1]]] << 2)
                            orow[12] = code
                            ev = [EV_NP, order[0], order[1], int(orow[3]), -1, -1, code, 0]
                        else:
                            ev = [EV_ABS2, order[0], order[1], int(orow[3]), -1, -1, 0, 0]
                    if is_block:
                        D = 1 << len(order)
                        orow[7] = em.n_slots
                        for _ in range(block_slots(D)):
                            em.new_slot()
                        orow[13] = D
                        em.blocks.append((list(op.factors), order, D, int(orow[7])))
                    elif adjoint and op.symbolic:
                        (gi,) = op.factors
                        info = infos[gi]
                        gm, _ = generator_matrix_from_terms(info.terms, order)
                        gm = gm * (2.0 * info.coeff)
                        orow[8] = len(em.genmats) // 2
                        em.genmats.extend(np.stack([gm.real, gm.imag], -1).reshape(-1).tolist())
                        orow[10] = _generator_kind(info.terms) if op.kind == OP_DENSE1 else \
                            (GK_P if orow[9] == CLS_NP else GK_MATRIX)
                        if orow[10] != GK_MATRIX:   # single Pauli: its scaled coefficient follows the matrix
                            beta = sum(c for f, c in info.terms if f)
                            em.genmats.extend([2.0 * info.coeff * beta, 0.0])
                        mkey = None
                        if frame and MERGE_SLOTS and orow[9] in (CLS_NX, CLS_NY) and orow[10] != GK_MATRIX:
                            mkey = (info.sym, int(orow[10]), float(np.float32(em.genmats[-2])))
                        if mkey is not None and mkey in merge_heads:
                            orow[7] = merge_heads[mkey]
                            orow[14] = 2                 # member: adds into the head's slot
                        else:
                            orow[7] = em.new_slot()
                            em.grad_slots.setdefault(info.sym, []).append(int(orow[7]))
                            if mkey is not None:
                                merge_heads[mkey] = int(orow[7])
                                orow[14] = 1             # head of a (possibly single) group
                    if ev is not None:
                        ev[4] = int(orow[7])
                        if is_block:
                            ev[7] = block_slots(1 << len(order))   # slots sharing the scale m
                        elif orow[14]:
                            ev[7] = int(orow[14])                  # merged slot: 1 head, 2 member
                        events.append(ev)
                elif op.kind == OP_DIAG:
                    terms = [(phys_mask(m), i_, w_) for m, i_, w_ in em.diag_terms(op)]
                    b_, e_, g_ = em.emit_terms(terms, reg_glob)
                    orow[4], orow[5], orow[6] = b_, e_, g_
                    if adjoint and op.symbolic:
                        orow[7] = em.new_slot()
                        em.grad_slots.setdefault(op.sym, []).append(int(orow[7]))
                    if frame:
                        orow[11] = em.angle_col(2, 0, 0.0)
                        events.append([EV_DIAG, -1, -1, -1, int(orow[7]), int(orow[11]), 0, 0])
                elif op.kind == OP_OBS:
                    obs = observables[op.obs]
                    terms = []
                    for ti, t in enumerate(obs.terms):
                        xm, zm, ny = term_masks(t)
                        assert xm == 0
                        terms.append((phys_mask(zm), -1 - em.n_coef, 0.0))  # negative: coefficient column
                        em.coef_cols.append((op.obs, ti))
                        em.n_coef += 1
                    b_, e_, g_ = em.emit_terms(terms, reg_glob)
                    orow[4], orow[5], orow[6] = b_, e_, g_
                    orow[7] = em.new_slot()
                    if adjoint:
                        em.energy_slots.append(int(orow[7]))
                    else:
                        em.obs_slots.setdefault(op.obs, []).append(int(orow[7]))
                    if frame:
                        orow[11] = em.angle_col(2, 0, 0.0)
                        events.append([EV_OBS, -1, -1, -1, int(orow[7]), int(orow[11]), 0, 0])
                em.op_rows.append(orow)
            srow[49] = len(em.op_rows)
            # tensor-core stage (forward, 16 amplitudes x 128 threads per tile, plan-specialised):
            # all of the stage's ops are full dense matrices on its register slots, so their product
            # is one 16 x 16 unitary per row, applied by tcgen05 MMAs (csrc/qf_tc.cu, jit.py)
            if tc_ok:
                rows_ = em.op_rows[int(srow[48]):int(srow[49])]
                dense = [r_ for r_ in rows_ if int(r_[0]) in (OP_DENSE1, OP_DENSE2)]
                cost = sum(4 if int(r_[0]) == OP_DENSE1 else 8 for r_ in dense)
                if (len(dense) == len(rows_) and cost >= TC_MIN_FFMA2 and
                        all(int(r_[9]) in (CLS_GENERAL, CLS_XLIKE, CLS_REAL) for r_ in dense)):
                    srow[50] = len(em.tc_blocks) + 1
                    em.tc_blocks.append([(int(r_[0]), int(r_[3]), int(r_[1]), int(r_[2])) for r_ in dense])
            em.stage_rows.append(srow)
        if frame and not adjoint:
            events.append([EV_PASS, -1, -1, -1, -1, -1, fwd_index, 0])
        prow[1] = len(em.stage_rows)
        prow[5] = em.n_mat
        prow[7] = em.n_ang
        prow[9] = em.n_slots
        prow[12] = em.n_coef
        prow[15] = len(em.term_mask)
        prow[81] = len(em.grp)
        prow[83] = len(em.op_rows)
        em.pass_rows.append(prow)

    # block-fused adjoint: one matrix per factor (embedded in the block's basis), allocated
    # after every pass's range so the pass kernels never stage them
    blocks, bfac, bgen = [], [], []
    for factors, order, D, slot0 in em.blocks:
        fb = len(bfac)
        for gi in factors:
            info = infos[gi]
            moff = em.dense_mat(Op(OP_DENSE1 if D == 2 else OP_DENSE2, tuple(order), factors=[gi]), order)
            goff, sym = -1, -1
            if info.symbolic:
                gm, _ = generator_matrix_from_terms(info.terms, order)
                gm = gm * (2.0 * info.coeff)
                goff = len(bgen) // 2
                bgen.extend(np.stack([gm.real, gm.imag], -1).reshape(-1).tolist())
                sym = info.sym
            bfac.append((moff, goff, sym))
        blocks.append((fb, len(bfac), D, slot0))

    # build recipe arrays
    gen_sym = np.array([g.sym for g in gen_rows], dtype=np.int32)
    gen_coeff = np.array([g.coeff for g in gen_rows], dtype=np.float64)
    gen_const = np.array([g.const for g in gen_rows], dtype=np.float64)
    gen_dim = np.array([1 << len(g.targets) for g in gen_rows], dtype=np.int32)
    gen_eval = np.zeros((len(gen_rows), 4))
    gen_evec = np.zeros((len(gen_rows), 4, 4), dtype=np.complex128)
    for k, g in enumerate(gen_rows):
        h = np.zeros((1 << len(g.targets),) * 2, dtype=np.complex128)
        for f, c in g.terms:
            h += _pauli_local(f, c, g.targets)
        w, v = np.linalg.eigh(h)
        d = len(w)
        gen_eval[k, :d] = w
        gen_evec[k, :d, :d] = v
    fbeg = [0]
    flat = []
    dmat, ddim = [], []
    for off, d, facs in em.dense_recipe:
        dmat.append(off)
        ddim.append(d)
        for f in facs:
            flat.extend(f)
        fbeg.append(len(flat) // 3)
    tsrc = np.array([(k, s) for k, s, _ in em.term_src], dtype=np.int32).reshape(-1, 2)
    tbeta = np.array([b for _, _, b in em.term_src], dtype=np.float64)
    recipe = dict(
        gen_sym=gen_sym, gen_coeff=gen_coeff, gen_const=gen_const, gen_dim=gen_dim,
        gen_eval=gen_eval.reshape(-1), gen_evec=np.stack([gen_evec.real, gen_evec.imag], -1).reshape(-1),
        n_fixed=n_fixed, n_const=n_const,
        dense_mat=np.array(dmat, dtype=np.int32), dense_dim=np.array(ddim, dtype=np.int32),
        dense_fbeg=np.array(fbeg, dtype=np.int32), factor=np.array(flat, dtype=np.int32),
        term_src=tsrc.reshape(-1), term_beta=tbeta,
    )
    stats = dict(passes=len(passes), stages=len(em.stage_rows), ops=len(em.op_rows), remapped=bool(remap),
                 stages_per_pass=[len(p.stages) for p in passes],
                 ops_per_pass=[len(p.ops) for p in passes], product_init=len(init),
                 tile_qubits=[p.qubits for p in passes],
                 lane_ops=sum(len(st.lane) for p in passes for st in p.stages))
    return Program(
        n=n, L=L, R=R, adjoint=adjoint,
        passes=np.array(em.pass_rows, dtype=np.int32).reshape(-1, PASS_INTS),
        stages=np.array(em.stage_rows, dtype=np.int32).reshape(-1, STAGE_INTS),
        ops=np.array(em.op_rows, dtype=np.int32).reshape(-1, OP_INTS),
        term_mask=np.array(em.term_mask, dtype=np.uint32),
        term_idx=np.array(em.term_idx, dtype=np.int32),
        term_w=np.array(em.term_w, dtype=np.float32),
        grp=np.array(em.grp, dtype=np.int32),
        genmats=np.array(em.genmats, dtype=np.float32),
        n_slots=em.n_slots, n_mat=em.n_mat, n_ang=em.n_ang, n_coef=em.n_coef,
        recipe=recipe, grad_slots=em.grad_slots, obs_slots=em.obs_slots,
        energy_slots=em.energy_slots, stats=stats, frame=frame,
        frame_events=np.array(events, dtype=np.int32).reshape(-1, EV_INTS),
        blocks=np.array(blocks, dtype=np.int32).reshape(-1, 4),
        block_factors=np.array(bfac, dtype=np.int32).reshape(-1, 3),
        block_gens=np.array(bgen, dtype=np.float64),
        final_pos=final_pos if remap else None,
        tc_blocks=em.tc_blocks or None,
    )


def _generator_kind(terms) -> int:
    plain = [(f, c) for f, c in terms if f]
    if len(plain) != 1 or len(plain[0][0]) != 1:
        return GK_MATRIX
    return {"X": GK_X, "Y": GK_Y, "Z": GK_Z}[next(iter(plain[0][0].values()))]


_PAULI = {
    "X": np.array([[0, 1], [1, 0]], dtype=np.complex128),
    "Y": np.array([[0, -1j], [1j, 0]], dtype=np.complex128),
    "Z": np.array([[1, 0], [0, -1]], dtype=np.complex128),
    "I": np.eye(2, dtype=np.complex128),
}


def _pauli_local(factors, coef, order):
    m = np.array([[coef]], dtype=np.complex128)
    for q in order:
        m = np.kron(m, _PAULI[factors.get(q, "I")])
    return m


def generator_matrix_from_terms(terms, order):
    """(non-identity part of the generator in local basis ``order``, identity coefficient)."""
    d = 1 << len(order)
    h = np.zeros((d, d), dtype=np.complex128)
    ident = 0.0
    for f, c in terms:
        if not f:
            ident += c
        else:
            h += _pauli_local(f, c, order)
    return h, ident


# ---------------------------------------------------------------------------
# per-row values of concrete gates
# ---------------------------------------------------------------------------

_MAT_CACHE: dict = {}


def concrete_matrix(g) -> np.ndarray:
    hit = _MAT_CACHE.get(id(g))
    if hit is not None and hit[0] is g:
        return hit[1]
    m = np.asarray(gate_matrix(g), dtype=np.complex128)
    if len(_MAT_CACHE) > 200_000:
        _MAT_CACHE.clear()
    _MAT_CACHE[id(g)] = (g, m)
    return m


def concrete_tables(circuits, infos):
    """fixed [Bf, n_fixed, 16] complex128 (4x4-stride) and const angles [Bc, n_const]."""
    fixed_pos = [i for i in infos if not i.symbolic and not i.diag]
    diag_pos = [i for i in infos if not i.symbolic and i.diag]
    n_fixed = len(fixed_pos)
    n_const = sum(1 << len(i.targets) for i in diag_pos)
    shared = all(c is circuits[0] for c in circuits) or len(circuits) == 1
    if not shared:
        shared = True
        for info in fixed_pos + diag_pos:
            g0 = circuits[0].gates[info.index]
            if any(c.gates[info.index] is not g0 for c in circuits[1:]):
                shared = False
                break
    rows = circuits[:1] if shared else circuits
    fixed = np.zeros((len(rows), max(n_fixed, 1), 4, 4), dtype=np.complex128)
    consts = np.zeros((len(rows), max(n_const, 1)), dtype=np.float64)
    for r, c in enumerate(rows):
        for info in fixed_pos:
            m = concrete_matrix(c.gates[info.index])
            d = m.shape[0]
            fixed[r, info.fixed, :d, :d] = m
        for info in diag_pos:
            m = concrete_matrix(c.gates[info.index])
            k = len(info.targets)
            consts[r, info.const_col:info.const_col + (1 << k)] = _walsh_angles(np.diag(m))
    return fixed, consts
