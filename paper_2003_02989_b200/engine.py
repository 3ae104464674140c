"""Batched execution engine: plan cache, device programs, and the call sequence
(build ops -> forward passes -> expectations -> adjoint passes -> slot reductions).

Everything numeric runs in libqfb200.so kernels on the current CUDA stream; torch
is used for device allocation and host<->device copies only.
"""

from __future__ import annotations

import ctypes as C
import itertools
import os
import threading
from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from . import planner as pl
from .circuit import circuit_symbols
from .pauli import as_pauli_sum, term_masks


def _require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2003_02989_b200 needs a CUDA device (B200, sm_100a); no CPU fallback exists")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    return dev


_TOTAL_MEM: dict = {}


def _total_memory(device) -> int:
    idx = device.index or 0
    if idx not in _TOTAL_MEM:
        _TOTAL_MEM[idx] = torch.cuda.get_device_properties(idx).total_memory
    return _TOTAL_MEM[idx]


class UniformBatch(list):
    """B rows of ONE circuit object (what ``ops.*`` build when a single circuit is passed):
    binding skips the per-row identity scans (the parameter-shift path binds 2*K*B rows)."""

    def __init__(self, circuit, rows: int):
        super().__init__([circuit] * rows)
        self.circuit = circuit


def _uniform(circuits) -> bool:
    return isinstance(circuits, UniformBatch)


def _ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


class DeviceProgram:
    """A planner.Program uploaded to one device + its ctypes descriptor."""

    def __init__(self, prog: pl.Program, device: torch.device):
        self.prog = prog
        self.device = device

        def up(a, dtype):
            a = np.ascontiguousarray(a)
            if a.size == 0:
                a = np.zeros(1, dtype=a.dtype)
            return torch.from_numpy(a).to(device=device, dtype=dtype)

        self.t_passes = up(prog.passes, torch.int32)
        self.t_stages = up(prog.stages, torch.int32)
        self.t_ops = up(prog.ops, torch.int32)
        self.t_mask = up(prog.term_mask.view(np.int32), torch.int32)
        self.t_idx = up(prog.term_idx, torch.int32)
        self.t_w = up(prog.term_w, torch.float32)
        self.t_grp = up(prog.grp, torch.int32)
        self.t_gen = up(prog.genmats, torch.float32)
        self.h_passes = np.ascontiguousarray(prog.passes)
        self.struct = nat.QfProgram(
            passes=_ptr(self.t_passes), stages=_ptr(self.t_stages), ops=_ptr(self.t_ops),
            term_mask=_ptr(self.t_mask), term_idx=_ptr(self.t_idx), term_w=_ptr(self.t_w),
            grp=_ptr(self.t_grp), genmats=_ptr(self.t_gen),
            n_passes=len(prog.passes), n_slots=prog.n_slots, n_mat=prog.n_mat, n_ang=prog.n_ang,
            n_coef=prog.n_coef, L=prog.L, R=prog.R, coef_row_stride=0,
            host_passes=self.h_passes.ctypes.data,
        )
        r = prog.recipe
        self.r_arrays = {k: up(v, _TORCH_OF[np.asarray(v).dtype]) for k, v in r.items()
                         if isinstance(v, np.ndarray)}
        self.n_gen = len(r["gen_sym"])
        self.n_fixed = r["n_fixed"]
        self.n_const = r["n_const"]
        self.n_dense = len(r["dense_mat"])
        self.max_dim = int(max(r["dense_dim"])) if len(r["dense_dim"]) else 0
        self.n_terms = len(r["term_beta"])
        self.tiles = 1 << (prog.n - prog.L)
        self._jit = None
        self._jit_cm = None
        self.frame = bool(prog.frame)
        ev = prog.frame_events if prog.frame_events is not None else np.zeros((0, pl.EV_INTS), np.int32)
        self.n_events = int(ev.shape[0])
        self.t_events = up(ev.reshape(-1), torch.int32)
        # slab prefix the frame walk touches (block factor matrices are allocated after it)
        span = [int(e[3]) + (16 if int(e[0]) in (pl.EV_ABS2, pl.EV_NP) else 4)
                for e in ev if int(e[0]) in (pl.EV_NX, pl.EV_NY, pl.EV_ABS1, pl.EV_ABS2, pl.EV_NP)]
        self.n_stage = min(max(span, default=1), max(prog.n_mat, 1))
        # tensor-core stages: recipe of every block's 16 x 16 product (qf_tc_build)
        self.n_tc = len(prog.tc_blocks or [])
        if self.n_tc:
            flat, ptr_ = [], [0]
            for blk_ in prog.tc_blocks:
                for kind_, moff_, s0_, s1_ in blk_:
                    flat.append((1 if kind_ == pl.OP_DENSE1 else 2, moff_, s0_, s1_))
                ptr_.append(len(flat))
            self.t_tc_ops = up(np.array(flat, dtype=np.int32).reshape(-1), torch.int32)
            self.t_tc_ptr = up(np.array(ptr_, dtype=np.int32), torch.int32)
        # block-fused adjoint: A slots reduced into consecutive columns, one range per block
        blk = prog.blocks if prog.blocks is not None else np.zeros((0, 4), np.int32)
        self.n_blocks = int(blk.shape[0])
        if self.n_blocks:
            blk = blk.copy()
            amap, col = {}, 0
            for i in range(self.n_blocks):
                D, slot0 = int(blk[i, 2]), int(blk[i, 3])
                for e in range(pl.block_slots(D)):
                    amap[col + e] = [slot0 + e]
                blk[i, 3] = col
                col += pl.block_slots(D)
            self.n_acols = col
            self.acsr = self.csr(amap, col)
            self.t_blocks = up(blk.reshape(-1), torch.int32)
            self.t_bfac = up(prog.block_factors.reshape(-1), torch.int32)
            self.t_bgen = up(prog.block_gens, torch.float64)
            self.n_bfac = int(prog.block_factors.shape[0])

    def recipe(self, fixed_t, fixed_rows, const_t, const_rows) -> nat.QfBuildRecipe:
        a = self.r_arrays
        return nat.QfBuildRecipe(
            n_gen=self.n_gen, gen_sym=_ptr(a["gen_sym"]), gen_coeff=_ptr(a["gen_coeff"]),
            gen_const=_ptr(a["gen_const"]), gen_dim=_ptr(a["gen_dim"]), gen_eval=_ptr(a["gen_eval"]),
            gen_evec=_ptr(a["gen_evec"]), n_fixed=max(self.n_fixed, 1), fixed=_ptr(fixed_t),
            fixed_rows=fixed_rows, n_dense=self.n_dense, dense_mat=_ptr(a["dense_mat"]),
            dense_dim=_ptr(a["dense_dim"]), dense_fbeg=_ptr(a["dense_fbeg"]), factor=_ptr(a["factor"]),
            n_terms=self.n_terms, term_src=_ptr(a["term_src"]), term_beta=_ptr(a["term_beta"]),
            term_const=_ptr(const_t), const_rows=const_rows, n_const=max(self.n_const, 1),
            max_dim=self.max_dim,
        )

    def jit(self, device, rows: int, force: bool = False):
        """Plan-specialised kernels for this program (compiled on first use) or None."""
        from . import jit as _jit

        # lane ops (warp-shuffle rotations) exist only in the plan-specialised kernels
        if not force and not _jit.enabled(rows, self.prog.n) and not self.prog.stats.get("lane_ops"):
            return None
        if self._jit_cm is None and _jit.CTAU and self.prog.adjoint:
            # adjoint programs: rotation coefficients from constant slabs (jit.CTAU) when the
            # launch's rows fit them; other row counts take the shared-memory variant
            with _JIT_LOCK:
                if self._jit_cm is None:
                    self._jit_cm = _jit.JitProgram(self.prog, device.index or 0, cm=True)
        if self._jit_cm is not None and self._jit_cm.cm and rows <= self._jit_cm.cm_rows_max:
            return self._jit_cm
        if self._jit_cm is not None and not self._jit_cm.cm:
            return self._jit_cm     # no rotation coefficients: the same kernels
        if self._jit is None:
            with _JIT_LOCK:
                if self._jit is None:
                    self._jit = _jit.JitProgram(self.prog, device.index or 0)
        return self._jit

    def csr(self, mapping: dict, n_cols: int):
        ptr = [0]
        lst = []
        for c in range(n_cols):
            lst.extend(mapping.get(c, []))
            ptr.append(len(lst))
        return (torch.tensor(ptr, dtype=torch.int32, device=self.device),
                torch.tensor(lst or [0], dtype=torch.int32, device=self.device))


_JIT_LOCK = threading.Lock()
# CUDA graphs of Bound.execute (QF_GRAPH=0 disables): (bound id, stream, want_grad, want_expect,
# theta shape) -> (bound, graph, static theta, static outputs); LRU-bounded because every graph
# keeps its buffers (the checkpointed adjoint's state copies) allocated
# Measured: headline e2e 20.67k -> 20.78k circuits/s; cfg1 (1024 x 2^10) 0.49 -> 0.53 ms (the
# replay's input copy and output clones outweigh 18 launches there) -> batches of at least
# GRAPH_MIN_AMPS amplitudes only
FRAME_MIN_AMPS = int(os.environ.get("QF_FRAME_MIN", str(1 << 24)))
GRAPHS = os.environ.get("QF_GRAPH", "1") not in ("0", "", "false")
MAX_GRAPHS = int(os.environ.get("QF_MAX_GRAPHS", "2"))
GRAPH_MIN_AMPS = 1 << 22
_GRAPHS: OrderedDict = OrderedDict()
_GRAPH_TOKENS = itertools.count(1)
_GRAPH_LOCK = threading.RLock()

_TORCH_OF = {
    np.dtype(np.int32): torch.int32, np.dtype(np.float64): torch.float64,
    np.dtype(np.float32): torch.float32, np.dtype(np.int64): torch.int64,
}


@dataclass
class ObsInfo:
    """Observables split into exact identity constants, fused diagonal ones and generic ones."""
    sums: list
    ident: np.ndarray                 # [n_obs] identity coefficient
    diag_ids: list
    generic_ids: list
    key: tuple = ()


def analyse_observables(observables, keep_identity: bool = False) -> ObsInfo:
    """``keep_identity``: identity terms stay in the (diagonal) observable and are weighted by
    the state norm -- used for shards of a distributed state, whose norms are not 1."""
    sums = [as_pauli_sum(o) for o in observables]
    ident = np.zeros(len(sums))
    stripped = []
    diag_ids, generic_ids = [], []
    for k, s in enumerate(sums):
        terms = []
        for t in s.terms:
            if not t.factors and not keep_identity:
                ident[k] += t.coefficient
            else:
                terms.append(t)
        stripped.append(terms)
        if terms and all(term_masks(t)[0] == 0 for t in terms):
            diag_ids.append(k)
        elif terms:
            generic_ids.append(k)
    key = tuple(tuple(tuple(sorted(t.factors.items())) for t in stripped[k]) for k in diag_ids)
    return ObsInfo(stripped, ident, diag_ids, generic_ids, key)


@dataclass
class Plan:
    n: int
    n_eff: int
    S: int
    infos: list
    fwd: DeviceProgram
    adj: DeviceProgram | None = None
    lam_diag: bool = False
    obs: ObsInfo | None = None
    extra: dict = field(default_factory=dict)


class Bound:
    """Everything of a batched call that does not depend on the symbol values:
    plan, concrete-gate tables, observable coefficient tables and reduction maps,
    all resident on the device.  ``execute`` then only launches kernels."""

    def __init__(self, engine, circuits, symbol_names, observables, want_grad, device, from_state=False,
                 want_state=False, norm_identity=False):
        self.device = device
        self.from_state = from_state
        self.symbol_names = list(symbol_names)
        sym_index = {s: i for i, s in enumerate(self.symbol_names)}
        uniform = _uniform(circuits)
        self.circuits = circuits if uniform else list(circuits)
        template = self.circuits[0]
        seen = set()
        for c in ((template,) if uniform else self.circuits):
            if id(c) in seen:
                continue
            seen.add(id(c))
            if c.num_qubits != template.num_qubits:
                raise pl.TopologyMismatch("all circuits of a batch must have the same register size")
            for s in circuit_symbols(c):
                if s not in sym_index:
                    raise KeyError(f"missing binding for symbol '{s}'")
        n = template.num_qubits
        if n > 32:
            raise MemoryError(f"{n} qubits exceeds the engine limit of 32 per device")
        self.obs = obs = analyse_observables(observables, keep_identity=norm_identity)
        self.n_obs = len(obs.sums)
        self.S = len(self.symbol_names)
        self.want_grad = want_grad
        # weighted Hamiltonian structure for the adjoint: H_b = sum_k up[b,k] obs_k
        self.lam_diag = False
        self.hkeys = []
        if want_grad:
            uniq: dict = {}
            for k, terms in enumerate(obs.sums):
                for t in terms:
                    uniq.setdefault(tuple(sorted(t.factors.items())), []).append((k, t.coefficient))
            self.hkeys = list(uniq)
            M = np.zeros((max(self.n_obs, 1), max(len(self.hkeys), 1)))
            for j, kk in enumerate(self.hkeys):
                for k, c in uniq[kk]:
                    M[k, j] += c
            self.hmix = torch.from_numpy(M).to(device)
            # weights of the default upstream (all ones): H_b = sum_k obs_k for every row
            self.hw_ones = torch.from_numpy(M.sum(axis=0, keepdims=True)).to(
                device=device, dtype=torch.float32).expand(len(self.circuits), M.shape[1]).contiguous()
            self.lam_diag = bool(self.hkeys) and all(all(p == "Z" for _, p in kk) for kk in self.hkeys)
        # Pauli-frame normalisation (planner.build_program): only where every output is a
        # diagonal observable / adjoint gradient and the plan-specialised kernels run
        from . import jit as _jit

        frame = (os.environ.get("QF_FRAME", "1") not in ("0", "", "false") and not want_state
                 and bool(obs.diag_ids) and not obs.generic_ids and (not want_grad or self.lam_diag)
                 and _jit.enabled(len(self.circuits), max(n, pl.N_MIN)))
        if frame and "QF_FRAME" not in os.environ and "QF_JIT" not in os.environ and \
                len(self.circuits) << max(n, pl.N_MIN) < FRAME_MIN_AMPS:
            # the frame walk (one thread per row, sequential over the gates) costs a fixed
            # ~0.1 ms; below 2^24 amplitudes it outweighs the FFMA2s it saves (cfg1 adjoint,
            # 1024 x 2^10: 0.45 -> 0.31 ms without)
            frame = False
        over = pl.batch_overrides(template, self.circuits, sym_index, pl.analyse(template, sym_index)) \
            if len(self.circuits) > 1 and not uniform else {}
        # block-fused adjoint (planner.build_ops(block=True)): plan-specialised kernels only
        jit_on = _jit.enabled(len(self.circuits), max(n, pl.N_MIN))
        block = (want_grad and os.environ.get("QF_BLOCK_ADJ", "1") not in ("0", "", "false") and jit_on)
        self.plan = engine.plan(template, sym_index, obs, want_grad, self.lam_diag,
                                tuple(self.hkeys) if want_grad else None, device, from_state, frame, over,
                                block=block, jit=jit_on)
        plan = self.plan
        self.frame = plan.fwd.frame

        fixed_np, const_np = pl.concrete_tables(self.circuits[:1] if uniform else self.circuits, plan.infos)
        self.fixed_rows, self.const_rows = fixed_np.shape[0], const_np.shape[0]
        self.fixed_t = torch.from_numpy(fixed_np.view(np.float64)).to(device)
        self.const_t = torch.from_numpy(const_np).to(device)
        if plan.adj is not None:
            infos_a = plan.extra["adj_infos"]
            fa, ca = pl.concrete_tables(self.circuits[:1] if uniform else self.circuits, infos_a)
            self.fixed_a = torch.from_numpy(fa.view(np.float64)).to(device)
            self.const_a = torch.from_numpy(ca).to(device)
            self.fixed_a_rows, self.const_a_rows = fa.shape[0], ca.shape[0]
        fw = plan.fwd
        coef_np = np.zeros(max(fw.prog.n_coef, 1), dtype=np.float32)
        col = 0
        for k in obs.diag_ids:
            for t in obs.sums[k]:
                coef_np[col] = t.coefficient
                col += 1
        self.fwd_coefs = torch.from_numpy(coef_np).to(device)
        self.obs_csr = fw.csr(fw.prog.obs_slots, self.n_obs)
        self.ident = torch.from_numpy(obs.ident).to(device)
        # generic (non-diagonal) observables
        self.gen_T = 0
        if obs.generic_ids:
            xs, zs, ys, cs, owner = [], [], [], [], []
            for k in obs.generic_ids:
                for t in obs.sums[k]:
                    xm, zm, ny = term_masks(t)
                    xs.append(xm); zs.append(zm); ys.append(ny); cs.append(t.coefficient); owner.append(k)
            self.gen_T = len(xs)
            self.gen_arrays = (torch.tensor(np.array(xs, dtype=np.uint32).view(np.int32), device=device),
                               torch.tensor(np.array(zs, dtype=np.uint32).view(np.int32), device=device),
                               torch.tensor(ys, dtype=torch.int32, device=device),
                               torch.tensor(cs, dtype=torch.float32, device=device))
            mapping: dict = {}
            for j, k in enumerate(owner):
                mapping.setdefault(k, []).append(j)
            self.gen_csr = fw.csr(mapping, self.n_obs)
        if want_grad:
            ad = plan.adj
            self.grad_csr = ad.csr(ad.prog.grad_slots, self.S)
            if ad.n_blocks:
                fmap: dict = {}
                for f, sym in enumerate(ad.prog.block_factors[:, 2].tolist()):
                    if sym >= 0:
                        fmap.setdefault(sym, []).append(f)
                self.block_csr = ad.csr(fmap, self.S)
            self.energy_csr = ad.csr({0: ad.prog.energy_slots}, 1)
            if not self.lam_diag and self.hkeys:
                xs, zs, ys = [], [], []
                for kk in self.hkeys:
                    xm, zm, ny = term_masks(_Term(dict(kk), 1.0))
                    xs.append(xm); zs.append(zm); ys.append(ny)
                self.h_arrays = (torch.tensor(np.array(xs, dtype=np.uint32).view(np.int32), device=device),
                                 torch.tensor(np.array(zs, dtype=np.uint32).view(np.int32), device=device),
                                 torch.tensor(ys, dtype=torch.int32, device=device))

    @property
    def B(self):
        return len(self.circuits)

    def execute(self, theta: torch.Tensor, *, upstream=None, want_state=False, want_grad=False,
                want_expect=True, stream=None, initial=None, donate=False, remote=None) -> dict:
        """theta: device float32 [B, S]; initial: [B, 2^n] complex state when bound
        ``from_state`` (the circuit is applied to it instead of |0...0>; ``donate``: the
        caller's contiguous complex64 device tensor is updated in place).  Returns device tensors.

        The common call (expectations / gradients of |0...0> programs, default upstream, the
        caller's current stream) replays a CUDA graph of the whole launch sequence (builds,
        frame walks, pass kernels, reductions: ~18 launches) captured on its first use."""
        if (GRAPHS and stream is None and upstream is None and initial is None and remote is None
                and not self.from_state and not want_state and theta.is_cuda
                and self.B << self.plan.n_eff >= GRAPH_MIN_AMPS):
            return self._execute_graphed(theta, want_grad, want_expect)
        return self._execute(theta, upstream=upstream, want_state=want_state, want_grad=want_grad,
                             want_expect=want_expect, stream=stream, initial=initial, donate=donate, remote=remote)

    def _execute_graphed(self, theta, want_grad, want_expect):
        dev = self.device
        cur = torch.cuda.current_stream(dev)
        theta = theta.to(dtype=torch.float32)
        key = (id(self), cur.cuda_stream, bool(want_grad), bool(want_expect), tuple(theta.shape))
        with _GRAPH_LOCK:
            hit = _GRAPHS.get(key)
            if hit is not None and hit[0] is self:
                _GRAPHS.move_to_end(key)
            else:
                from . import jit as _jit

                if hit is not None:                    # a dead Bound's graph under a reused id
                    stale = _GRAPHS.pop(key)
                    torch.cuda.synchronize(dev)
                    stale[1].reset()
                    _jit.release_slab_owner(stale[4])
                static = torch.empty(theta.shape, dtype=torch.float32, device=dev)
                static.copy_(theta)

                side = torch.cuda.Stream(dev)
                side.wait_stream(cur)
                graph = torch.cuda.CUDAGraph()
                # the graph owns its copies of the kernel modules with constant slabs (jit.CTAU):
                # loaded by the warm-up, written only by this graph's own replays, pinned until
                # the graph leaves the cache
                token = next(_GRAPH_TOKENS)
                with _jit.slab_owner(token):
                    with torch.cuda.stream(side):      # warm-up: NVRTC compiles, allocator sizing
                        self._execute(static, want_grad=want_grad, want_expect=want_expect)
                    cur.wait_stream(side)
                    with torch.cuda.graph(graph, stream=side, capture_error_mode="thread_local"):
                        out = self._execute(static, want_grad=want_grad, want_expect=want_expect)
                hit = (self, graph, static, out, token)
                _GRAPHS[key] = hit
                while len(_GRAPHS) > MAX_GRAPHS:       # each graph holds its buffers (checkpoints)
                    _, gone = _GRAPHS.popitem(last=False)
                    torch.cuda.synchronize(dev)
                    gone[1].reset()                    # the graph goes before its kernel modules
                    _jit.release_slab_owner(gone[4])
            _, graph, static, out, _ = hit
            static.copy_(theta, non_blocking=True)
            graph.replay()
            # outputs are copied before the lock is released: the next replay on this stream
            # rewrites the graph's static buffers
            return {k: (v.clone() if isinstance(v, torch.Tensor) else v) for k, v in out.items()}

    def _execute(self, theta: torch.Tensor, *, upstream=None, want_state=False, want_grad=False,
                 want_expect=True, stream=None, initial=None, donate=False, remote=None) -> dict:
        lib = nat.load()
        dev = self.device
        plan = self.plan
        B = self.B
        if stream is None:
            stream = torch.cuda.current_stream(dev).cuda_stream
        if theta.shape[1] == 0:
            theta = torch.zeros((B, 1), dtype=torch.float32, device=dev)
        fw = plan.fwd
        n_eff = plan.n_eff
        if self.from_state:
            if initial is None:
                raise ValueError("this binding applies the circuit to a given state: pass initial=")
            init = torch.as_tensor(initial).to(device=dev, dtype=torch.complex64).reshape(B, -1)
            if init.shape[1] != (1 << plan.n):
                raise ValueError(f"initial state has {init.shape[1]} amplitudes, expected {1 << plan.n}")
            if n_eff == plan.n:
                donated = donate and isinstance(initial, torch.Tensor) and initial.is_contiguous() and \
                    initial.dtype == torch.complex64 and initial.device == dev
                psi = init if donated else init.clone()  # kernels update psi in place
            else:
                psi = torch.zeros((B, 1 << n_eff), dtype=torch.complex64, device=dev)
                psi[:, : 1 << plan.n] = init
        else:
            psi = torch.empty((B, 1 << n_eff), dtype=torch.complex64, device=dev)
        mats = torch.empty((B, max(fw.prog.n_mat, 1)), dtype=torch.complex64, device=dev)
        angs = torch.empty((B, max(fw.prog.n_ang, 1)), dtype=torch.int32, device=dev)
        rec = fw.recipe(self.fixed_t, self.fixed_rows, self.const_t, self.const_rows)
        nat.check(lib.qf_build_ops(C.byref(rec), _ptr(theta), theta.shape[1], B, _ptr(mats), fw.prog.n_mat,
                                   _ptr(angs), fw.prog.n_ang, stream))
        scale = None
        ckpt = self._checkpoints(psi, want_grad and not want_state and remote is None)
        if fw.frame:
            if want_state:
                raise ValueError("this binding stores frame-normalised states (expectations / gradients "
                                 "only); bind with want_state=True for states")
            scale = torch.empty((B, max(fw.prog.n_slots, 1)), dtype=torch.float64, device=dev)
            frame_f = torch.empty((B, 2), dtype=torch.float64, device=dev)  # QfFrame {u32 x, z; f64 m}
            pm = (_ptr(ckpt[1]), ckpt[1].shape[1]) if ckpt else (None, 0)
            nat.check(lib.qf_frame_walk_ckpt(_ptr(fw.t_events), fw.n_events, 0, B, _ptr(mats), fw.prog.n_mat,
                                             _ptr(angs), fw.prog.n_ang, _ptr(scale), fw.prog.n_slots, None,
                                             _ptr(frame_f), pm[0], pm[1], fw.n_stage, stream))
        else:
            frame_f = None
        partials = torch.empty((B, max(fw.prog.n_slots, 1), fw.tiles), dtype=torch.float64, device=dev)
        # relabelled programs and tensor-core stages exist only as plan-specialised kernels; the
        # stages' B images are built from the (frame-walked) slab
        jf = fw.jit(dev, B, force=remote is not None or fw.prog.final_pos is not None or fw.n_tc > 0)
        tcb = None
        if fw.n_tc:
            tcb = torch.empty((B, fw.n_tc, 2048), dtype=torch.float32, device=dev)
            nat.check(lib.qf_tc_build(_ptr(mats), fw.prog.n_mat, B, _ptr(fw.t_tc_ops), _ptr(fw.t_tc_ptr), fw.n_tc,
                                      _ptr(tcb), stream))
        tck = dict(tcb=_ptr(tcb), tc_n=fw.n_tc)
        turn = self._turn() if ckpt else None
        prep = None
        if ckpt and turn is not None:
            # forward passes 0..P-2, then ONE kernel for the forward's last pass and the
            # backward's first (the final state stays in registers), then backward 1..P-1
            ck = ckpt[0]
            P = len(ck)
            prep = self._adjoint_prep(lib, psi, theta, upstream, stream, frame_f, ckpt)
            jf.run_ckpt(B, [_ptr(t) for t in ck], [0] + [_ptr(t) for t in ck[:-1]], 0, _ptr(mats), _ptr(angs),
                        _ptr(self.fwd_coefs), 0, _ptr(partials), stream, False, which=range(P - 1), **tck)
            hw_t = prep["hw_t"]
            turn.run(B, _ptr(ck[P - 2]), _ptr(mats), _ptr(angs), _ptr(self.fwd_coefs), _ptr(partials),
                     _ptr(prep["lam"]), _ptr(prep["mats"]), _ptr(prep["angs"]), _ptr(hw_t), hw_t.shape[1],
                     _ptr(prep["partials"]), stream)
            self._adjoint_launch(lib, prep, psi, stream, ckpt, first=1)
        elif ckpt:
            ck = ckpt[0]
            jf.run_ckpt(B, [_ptr(t) for t in ck], [0] + [_ptr(t) for t in ck[:-1]], 0, _ptr(mats), _ptr(angs),
                        _ptr(self.fwd_coefs), 0, _ptr(partials), stream, False, **tck)
        elif jf is not None:
            jf.run(B, _ptr(psi), 0, _ptr(mats), _ptr(angs), _ptr(self.fwd_coefs), 0, _ptr(partials), stream,
                   remote=remote, **tck)
        else:
            nat.check(lib.qf_run_passes(C.byref(fw.struct), 0, len(fw.prog.passes), _ptr(psi), n_eff, B,
                                        _ptr(mats), _ptr(angs), _ptr(self.fwd_coefs), _ptr(partials), fw.tiles,
                                        stream))
        out: dict = {}
        if self.n_obs and want_expect:
            # the diagonal reduction writes every column (empty columns get 0) plus the identity
            # constants: no zero-fill, no separate add
            expv = torch.empty((B, self.n_obs), dtype=torch.float64, device=dev)
            ptr, lst = self.obs_csr
            nat.check(lib.qf_reduce_slots_offset(_ptr(partials), B, fw.prog.n_slots, fw.tiles, _ptr(ptr),
                                                 _ptr(lst), self.n_obs, _ptr(expv), 0, _ptr(scale),
                                                 _ptr(self.ident), stream))
            if self.gen_T:
                xm, zm, ny, cf = self.gen_arrays
                chunks = ((1 << n_eff) + 2047) // 2048
                part = torch.empty((B, self.gen_T, chunks), dtype=torch.float64, device=dev)
                nat.check(lib.qf_pauli_expect(_ptr(psi), n_eff, B, self.gen_T, _ptr(xm), _ptr(zm), _ptr(ny),
                                              _ptr(cf), 0, _ptr(part), stream))
                ptr, lst = self.gen_csr
                nat.check(lib.qf_reduce_slots(_ptr(part), B, self.gen_T, chunks, _ptr(ptr), _ptr(lst), self.n_obs,
                                              _ptr(expv), 1, stream))
            out["expectations"] = expv
        if want_state:
            if fw.prog.final_pos is not None:
                # relabelled program: physical bit final_pos[q] holds qubit q -- one
                # device-side bit-permuting copy back to the logical layout
                psi = _unrelabel(psi, fw.prog.final_pos, n_eff)
            st = psi[:, : (1 << plan.n)]
            out["state"] = st.clone() if want_grad else st
        if want_grad:
            if prep is not None:      # the turn kernel already ran the backward sweep
                self._adjoint_reduce(lib, prep, stream, out)
            else:
                self._adjoint(lib, psi, theta, upstream, stream, out, frame_f, ckpt)
        return out

    def _checkpoints(self, psi, wanted):
        """Checkpointed adjoint (plan.extra["ckpt"]): the forward passes write every pass
        output to its own buffer, so the adjoint sweep reloads psi from them instead of
        un-applying and storing it -- one state write per backward pass fewer, and exact
        forward states.  Returns (buffers, pass scales [B, P]) or None when off / no room."""
        plan = self.plan
        if not (wanted and plan.extra.get("ckpt")):
            return None
        fw = plan.fwd
        P = len(fw.prog.passes)
        if fw.jit(self.device, self.B) is None or plan.adj.jit(self.device, self.B) is None:
            return None
        need = (P - 1) * psi.numel() * psi.element_size()
        # a static budget: cudaMemGetInfo stalls for up to tens of ms while kernels run
        if need > 0.3 * _total_memory(self.device):
            return None
        try:
            ck = [torch.empty_like(psi) for _ in range(P - 1)] + [psi]
        except torch.cuda.OutOfMemoryError:
            return None
        return ck, torch.empty((self.B, P), dtype=torch.float64, device=self.device)

    def _adjoint(self, lib, psi, theta, upstream, stream, out, frame_f=None, ckpt=None):
        prep = self._adjoint_prep(lib, psi, theta, upstream, stream, frame_f, ckpt)
        self._adjoint_launch(lib, prep, psi, stream, ckpt, first=0)
        self._adjoint_reduce(lib, prep, stream, out)

    def _adjoint_prep(self, lib, psi, theta, upstream, stream, frame_f=None, ckpt=None) -> dict:
        """Per-call tables of the backward sweep: Hamiltonian weights, built matrices / angles,
        the frame walk, lambda and the slot partials."""
        plan, dev, B = self.plan, self.device, self.B
        ad = plan.adj
        n_eff = plan.n_eff
        if upstream is None:
            hw_t = self.hw_ones   # precomputed at bind time: no per-step ATen work
        else:
            up = torch.as_tensor(upstream, dtype=torch.float64).to(dev).reshape(B, -1)
            if up.shape[1] != self.n_obs:
                raise ValueError(f"upstream shape {tuple(up.shape)} != ({B}, {self.n_obs})")
            # elementwise product + fixed-order sum: bit-identical across calls and threads (a
            # cuBLAS GEMM may pick different reduction orders)
            hw_t = (up[:, :, None] * self.hmix[None, :, :]).sum(dim=1).to(torch.float32).contiguous()
        mats = torch.empty((B, max(ad.prog.n_mat, 1)), dtype=torch.complex64, device=dev)
        angs = torch.empty((B, max(ad.prog.n_ang, 1)), dtype=torch.int32, device=dev)
        rec = ad.recipe(self.fixed_a, self.fixed_a_rows, self.const_a, self.const_a_rows)
        nat.check(lib.qf_build_ops(C.byref(rec), _ptr(theta), theta.shape[1], B, _ptr(mats), ad.prog.n_mat,
                                   _ptr(angs), ad.prog.n_ang, stream))
        scale = None
        if ad.frame:
            scale = torch.empty((B, max(ad.prog.n_slots, 1)), dtype=torch.float64, device=dev)
            pm = (_ptr(ckpt[1]), ckpt[1].shape[1]) if ckpt else (None, 0)
            nat.check(lib.qf_frame_walk_ckpt(_ptr(ad.t_events), ad.n_events, 1, B, _ptr(mats), ad.prog.n_mat,
                                             _ptr(angs), ad.prog.n_ang, _ptr(scale), ad.prog.n_slots, _ptr(frame_f),
                                             None, pm[0], pm[1], ad.n_stage, stream))
        lam = torch.empty_like(psi)
        partials = torch.empty((B, max(ad.prog.n_slots, 1), ad.tiles), dtype=torch.float64, device=dev)
        return dict(hw_t=hw_t, mats=mats, angs=angs, scale=scale, lam=lam, partials=partials)

    def _adjoint_launch(self, lib, prep, psi, stream, ckpt, first=0):
        """The backward pass kernels from pass ``first`` (1 after the turn kernel)."""
        plan, dev, B = self.plan, self.device, self.B
        ad = plan.adj
        n_eff = plan.n_eff
        hw_t, mats, angs, lam, partials = prep["hw_t"], prep["mats"], prep["angs"], prep["lam"], prep["partials"]
        if not self.lam_diag and first == 0:
            if self.hkeys:
                xm, zm, ny = self.h_arrays
                nat.check(lib.qf_pauli_apply(_ptr(psi), _ptr(lam), n_eff, B, len(self.hkeys), _ptr(xm), _ptr(zm),
                                             _ptr(ny), _ptr(hw_t), hw_t.shape[1], stream))
            else:
                lam.zero_()
        # block-fused and R = 5 adjoint programs exist only as plan-specialised kernels
        ja = ad.jit(dev, B, force=ad.n_blocks > 0 or ad.prog.R != pl.ADJ_R)
        if ckpt:
            ck = ckpt[0]
            ja.run_ckpt(B, [_ptr(t) for t in reversed(ck)], None, _ptr(lam), _ptr(mats), _ptr(angs), _ptr(hw_t),
                        hw_t.shape[1], _ptr(partials), stream, True, which=range(first, len(ck)))
        elif ja is not None:
            ja.run(B, _ptr(psi), _ptr(lam), _ptr(mats), _ptr(angs), _ptr(hw_t), hw_t.shape[1], _ptr(partials),
                   stream)
        else:
            struct = nat.QfProgram.from_buffer_copy(ad.struct)
            struct.coef_row_stride = hw_t.shape[1]
            nat.check(lib.qf_adjoint_passes(C.byref(struct), 0, len(ad.prog.passes), _ptr(psi), _ptr(lam), n_eff,
                                            B, _ptr(mats), _ptr(angs), _ptr(hw_t), _ptr(partials), ad.tiles,
                                            stream))

    def _adjoint_reduce(self, lib, prep, stream, out):
        plan, dev, B = self.plan, self.device, self.B
        ad = plan.adj
        mats, partials, scale = prep["mats"], prep["partials"], prep["scale"]
        # every column is written by the first reduction (S > 0)
        grad = torch.empty((B, self.S), dtype=torch.float64, device=dev) if self.S else \
            torch.zeros((B, 1), dtype=torch.float64, device=dev)
        if self.S:
            ptr, lst = self.grad_csr
            nat.check(lib.qf_reduce_slots_scaled(_ptr(partials), B, ad.prog.n_slots, ad.tiles, _ptr(ptr), _ptr(lst),
                                                 self.S, _ptr(grad), 0, _ptr(scale), stream))
        if ad.n_blocks and self.S:
            # fused blocks: reduce each block's A matrix, then every factor's gradient from it
            acols = torch.empty((B, ad.n_acols), dtype=torch.float64, device=dev)
            ptr, lst = ad.acsr
            nat.check(lib.qf_reduce_slots_scaled(_ptr(partials), B, ad.prog.n_slots, ad.tiles, _ptr(ptr), _ptr(lst),
                                                 ad.n_acols, _ptr(acols), 0, _ptr(scale), stream))
            vals = torch.empty((B, ad.n_bfac), dtype=torch.float64, device=dev)
            nat.check(lib.qf_block_grads(_ptr(ad.t_blocks), ad.n_blocks, _ptr(ad.t_bfac), ad.n_bfac, _ptr(ad.t_bgen),
                                         _ptr(mats), ad.prog.n_mat, _ptr(acols), ad.n_acols, _ptr(vals), B, stream))
            ptr, lst = self.block_csr
            nat.check(lib.qf_reduce_slots(_ptr(vals), B, ad.n_bfac, 1, _ptr(ptr), _ptr(lst), self.S, _ptr(grad), 1,
                                          stream))
        if self.lam_diag:
            energy = torch.empty((B, 1), dtype=torch.float64, device=dev)
            ptr, lst = self.energy_csr
            nat.check(lib.qf_reduce_slots_scaled(_ptr(partials), B, ad.prog.n_slots, ad.tiles, _ptr(ptr), _ptr(lst),
                                                 1, _ptr(energy), 0, _ptr(scale), stream))
            out["energy"] = energy[:, 0]
        out["grad"] = grad[:, : self.S]

    def _turn(self):
        """The turn kernel (jit.TurnKernel: forward's last pass + backward's first pass in one
        launch) for this plan, or None."""
        plan = self.plan
        if os.environ.get("QF_TURN", "1") in ("0", "", "false") or plan.adj is None:
            return None
        if "turn" not in plan.extra:
            from . import jit as _jit

            with _JIT_LOCK:
                if "turn" not in plan.extra:
                    ok = _jit._turn_compatible(plan.fwd.prog, plan.adj.prog)
                    plan.extra["turn"] = _jit.TurnKernel(plan.fwd.prog, plan.adj.prog,
                                                         self.device.index or 0) if ok else None
        return plan.extra["turn"]


def _obs_key(o) -> tuple:
    """Content key of an observable (terms and coefficients): callers that pass a fresh
    PauliString / reference PauliSum object per call still hit the binding cache."""
    s = as_pauli_sum(o)
    return tuple((tuple(sorted(t.factors.items())), float(t.coefficient)) for t in s.terms)


def _unrelabel(psi: torch.Tensor, final_pos, n: int) -> torch.Tensor:
    """[B, 2^n] state whose physical bit final_pos[q] is logical qubit q -> logical layout
    (one coalesced-write gather kernel, ``qf_permute_bits``)."""
    lib = nat.load()
    out = torch.empty_like(psi)
    pos = (C.c_int32 * n)(*[int(x) for x in final_pos])
    nat.check(lib.qf_permute_bits(_ptr(psi), _ptr(out), n, psi.shape[0], C.cast(pos, C.c_void_p),
                                  torch.cuda.current_stream(psi.device).cuda_stream))
    return out


class Engine:
    def __init__(self, max_bound: int = 64, max_plans: int = 256):
        self._plans: OrderedDict = OrderedDict()
        self._bound: OrderedDict = OrderedDict()
        self._max_bound = max_bound
        self._max_plans = max_plans
        self._lock = threading.Lock()

    def plan(self, template, symbol_index, obs: ObsInfo, adjoint: bool, lam_diag: bool, hkeys, device,
             from_state: bool = False, frame: bool = False, overrides=None, block: bool = False,
             jit: bool = False):
        overrides = overrides or {}
        topo = pl.topology_key(template, symbol_index)
        key = (topo, obs.key, tuple(obs.diag_ids), adjoint, lam_diag, hkeys, str(device), from_state, frame,
               tuple(sorted(overrides.items())), pl.FUSION_ENABLED, block, jit, pl.REMAP, pl.TC_STAGES,
               pl.LANE_OPS, pl.VEC_EDGE)
        with self._lock:
            hit = self._plans.get(key)
            if hit is not None:
                self._plans.move_to_end(key)
        if hit is not None:
            return hit
        n = template.num_qubits
        n_eff = max(n, pl.N_MIN)
        infos = pl.analyse(template, symbol_index, overrides)
        if frame and adjoint:  # forward and adjoint must agree on the stored representation
            frame = pl.frame_eligible(pl.build_ops(pl.analyse(template, symbol_index, overrides), True), infos, True)
        elif frame:
            # forward only: no normalisable rotation (HEA runs fused into general 1q matrices,
            # brickwork) -> no frame walk (it cost as much as the passes in cfg1's shifted batches)
            frame = pl.has_normalisable(pl.build_ops(pl.analyse(template, symbol_index, overrides), False), infos)
        diag_sums = [None] * len(obs.sums)
        for k in obs.diag_ids:
            diag_sums[k] = _TermList(obs.sums[k])
        adjp = None
        if adjoint:
            infos_a = pl.analyse(template, symbol_index, overrides)
            hterms = _TermList([_Term(dict(kk), 1.0) for kk in hkeys])
            adjp = pl.build_program(template, infos_a, n_eff, adjoint=True, observables=[hterms],
                                    lam_diag=lam_diag, frame=frame, block=block, jit=jit)
        ckpt = False
        if adjp is not None and frame and lam_diag and not from_state and \
                os.environ.get("QF_CKPT", "1") not in ("0", "", "false"):
            fwd = pl.build_program(template, infos, n_eff, adjoint=False, observables=diag_sums,
                                   obs_diag_ids=obs.diag_ids, from_state=from_state, frame=frame, mirror=True,
                                   block=block, vec=jit)
            # the adjoint's backward pass i must undo exactly forward pass P-1-i (both lists
            # are in forward order), and both frame walks must hold the same Pauli frame at every
            # pass boundary: true for normalised rotations and diagonal ops, not for general
            # dense ops (the forward absorbs the frame in front of them, the adjoint behind)
            ev = adjp.frame_events if adjp.frame_events is not None else np.zeros((0, pl.EV_INTS), np.int32)
            ckpt = (fwd.frame and adjp.frame and fwd.stats["tile_qubits"] == adjp.stats["tile_qubits"]
                    and fwd.stats["ops_per_pass"] == adjp.stats["ops_per_pass"]
                    and not np.isin(np.asarray(ev)[:, 0], (pl.EV_ABS1, pl.EV_ABS2)).any())
            if not ckpt:
                infos = pl.analyse(template, symbol_index, overrides)
        if not ckpt:
            # jit (qubit relabelling, planner.plan_passes_remap) only without a backward sweep,
            # which loads the forward's output in the identity layout
            fwd = pl.build_program(template, infos, n_eff, adjoint=False, observables=diag_sums,
                                   obs_diag_ids=obs.diag_ids, from_state=from_state, frame=frame,
                                   jit=jit and not adjoint, vec=jit)
        plan = Plan(n, n_eff, len(symbol_index), infos, DeviceProgram(fwd, device), None, lam_diag, obs)
        plan.extra["from_state"] = from_state
        plan.extra["ckpt"] = ckpt
        if adjp is not None:
            assert adjp.frame == fwd.frame
            plan.adj = DeviceProgram(adjp, device)
            plan.extra["adj_infos"] = infos_a
        with self._lock:
            self._plans[key] = plan
            while len(self._plans) > self._max_plans:   # LRU: device tables + NVRTC modules go with it
                self._plans.popitem(last=False)
        return plan

    def bind(self, circuits, symbol_names, observables=(), *, want_grad=False, device=None,
             from_state=False, want_state=False, norm_identity=False) -> Bound:
        dev = _require_cuda(device)
        symbol_names = tuple(s.name if hasattr(s, "name") else s for s in symbol_names)
        observables = list(observables)
        uniform = _uniform(circuits)
        ckey = ("uniform", id(circuits.circuit), len(circuits)) if uniform else tuple(map(id, circuits))
        key = (ckey, symbol_names, tuple(_obs_key(o) for o in observables), bool(want_grad), str(dev),
               bool(from_state), bool(want_state), bool(norm_identity), pl.FUSION_ENABLED, pl.REMAP,
               pl.TC_STAGES, pl.LANE_OPS, pl.VEC_EDGE)
        with self._lock:
            hit = self._bound.get(key)
            if hit is not None:
                self._bound.move_to_end(key)
        if hit is not None and (hit.circuits[0] is circuits[0] if uniform else
                                all(a is b for a, b in zip(hit.circuits, circuits))):
            return hit
        b = Bound(self, circuits, symbol_names, observables, want_grad, dev, from_state, want_state,
                  norm_identity)
        b._keepalive = observables
        with self._lock:
            if len(self._bound) >= self._max_bound:
                self._bound.popitem(last=False)
            self._bound[key] = b
        return b

    def run(self, circuits, symbol_names, values, observables=(), *, want_state=False, want_grad=False,
            upstream=None, device=None):
        """One-shot convenience: bind (cached) + execute.  values: [B, S]."""
        dev = _require_cuda(device)
        vals = values if isinstance(values, torch.Tensor) else torch.as_tensor(np.asarray(values, dtype=np.float32))
        if vals.ndim == 1:
            vals = vals.reshape(1, -1) if len(symbol_names) else vals.reshape(-1, 0)
        B = int(vals.shape[0])
        if not isinstance(circuits, (list, tuple)):
            circuits = [circuits] * B
        if len(circuits) != B:
            raise ValueError(f"{len(circuits)} circuits for {B} parameter rows")
        if B == 0:
            return {}
        bound = self.bind(circuits, symbol_names, observables, want_grad=want_grad, device=dev,
                          want_state=want_state)
        theta = vals.to(device=dev, dtype=torch.float32).contiguous()
        out = bound.execute(theta, upstream=upstream, want_state=want_state, want_grad=want_grad)
        out["plan"] = bound.plan
        return out


class _Term:
    __slots__ = ("factors", "coefficient")

    def __init__(self, factors, coefficient):
        self.factors = dict(factors)
        self.coefficient = coefficient


class _TermList:
    def __init__(self, terms):
        self.terms = list(terms.terms if hasattr(terms, "terms") else terms)


ENGINE = Engine()
