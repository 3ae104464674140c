"""Plan-specialised tile-pass kernels.

The interpreted ``qf::pass_kernel`` reads the program descriptors at run time; ncu
showed its cost is dominated by descriptor decode, op dispatch over many template
instantiations (instruction-cache misses) and per-op warp reductions, not by the
gate arithmetic.  This module emits, from exactly the same planner.Program, one
straight-line CUDA kernel per pass in which every register slot, matrix-class,
matrix offset, phase-polynomial mask and register subset, swizzled shared-memory
offset and gradient slot is a compile-time constant; libqfb200's ``qf_jit_*``
entry points compile it with NVRTC (sm_100a) and launch it.  Only per-row numbers
(gate matrices, angles, observable coefficients) are read at run time.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import os
import threading
import weakref

import numpy as np

from . import _native as nat
from . import planner as pl

_HERE = os.path.dirname(os.path.abspath(__file__))
_PRELUDE = None
_CACHE: dict = {}
_LOCK = threading.Lock()


def prelude() -> str:
    global _PRELUDE
    if _PRELUDE is None:
        with open(os.path.join(_HERE, "csrc", "qf_jit_prelude.cuh")) as f:
            _PRELUDE = f.read()
    return _PRELUDE


class QfJitArgs(C.Structure):
    _fields_ = [("psi", C.c_void_p), ("lam", C.c_void_p), ("mats", C.c_void_p), ("angles", C.c_void_p),
                ("coefs", C.c_void_p), ("partials", C.c_void_p), ("n_mat", C.c_int), ("n_ang", C.c_int),
                ("coef_stride", C.c_int), ("n_slots", C.c_int), ("tiles_log2", C.c_int), ("pad", C.c_int),
                ("peers", C.c_void_p), ("rank_base", C.c_int), ("pad2", C.c_int),
                ("psi_src", C.c_void_p), ("skip_psi", C.c_int), ("pad3", C.c_int),
                ("tcb", C.c_void_p), ("tc_n", C.c_int), ("pad4", C.c_int)]


# constant-bank rotation coefficients: a pass's staged matrix slab for every row of the launch
# is copied into a __constant__ array of its module (qf_cm_<tag>, [rows][mcnt] float2), so the
# Pauli-frame rotation coefficient tau is read with a uniform-register load (LDCU) and every
# rotation FFMA2 reads only two vector registers: an FP32x2 FMA with three fresh register
# sources issues once per 3 cycles instead of 2 (tools/micro/ffma2_bench.cu,
# tools/regread_model.py).  Used when rows * mcnt fits CM_CAP (JitProgram picks the variant).
CTAU = os.environ.get("QF_CTAU", "1") not in ("0", "", "false")
CM_CAP = 8192   # float2 entries: 64 KB, the __constant__ limit of a module
CM_MAX_COPIES = 16   # per-stream module copies of one program (graphs capture on their own stream)
FUSED_GRAD = os.environ.get("QF_FUSED_GRAD", "0") not in ("0", "", "false")   # measured 2% slower
CHUNKED_GS = os.environ.get("QF_CHUNKED_GS", "1") not in ("0", "", "false")
GS_THREAD_BYTES = int(os.environ.get("QF_GS_BYTES", str(40 * 1024)))
# 0: one CTA per tile; 1: persistent CTAs (measured slower); 2: persistent CTAs that prefetch
# the next tile into shared memory with cp.async while computing the current one
PERSIST_MODE = int(os.environ.get("QF_PERSIST", "0") or 0)
PERSIST = PERSIST_MODE > 0
# timing experiments only (results are WRONG): "noload" -- tiles start from register values
# derived from the thread index instead of global loads; "nocompute" -- stages do no gate
# arithmetic (exchanges, loads and stores stay); "memonly" -- loads and stores only
EXP_MODE = os.environ.get("QF_EXP", "")
# integer-weight phase tables: "f4" 16-byte entries (c, c, -s, s) -- no ALU work per lookup;
# (measured: "cs" is faster, forward middle passes 0.93 -> 0.86 ms on the headline)
# "cs" 8-byte (c, s) entries (half the shared-memory bytes, one FADD per lookup)
TB_MODE = os.environ.get("QF_TB_MODE", "cs")
# L2 prefetch of the tile the next wave of CTAs will load (cp.async.bulk.prefetch.L2, issued
# right after this tile's own loads): 0 off, 1 adjoint passes, 2 every pass
L2PF = int(os.environ.get("QF_L2PF", "0") or 0)
# a barrier before each inner exchange's writes (not needed: see generate)
PREW_SYNC = os.environ.get("QF_PREW_SYNC", "0") not in ("0", "", "false")
SPLIT_XCHG = os.environ.get("QF_SPLIT_XCHG", "0") not in ("0", "", "false")
# exchange addresses as (tp ^ low nibble) + high bits (immediate offsets; _sm_idx)
XADD = os.environ.get("QF_XADD", "1") not in ("0", "", "false")
GS_RING = int(os.environ.get("QF_GS_RING", "16"))
ADJ_LOADS_FIRST = os.environ.get("QF_ADJ_LOADS_FIRST", "auto")   # "0", "1" or "auto" (heavy passes)
SPLIT_LIGHT_OPS = int(os.environ.get("QF_SPLIT_LIGHT_OPS", "64"))
ADJ3 = os.environ.get("QF_ADJ3", "0") not in ("0", "", "false")
L2PF_SMS = int(os.environ.get("QF_L2PF_SMS", "148"))
# integer-weight phase polynomials evaluated per amplitude in Gray-code order (one live value)
# instead of by a 2^R-entry Walsh transform
# frame-normalised rotations of the adjoint take their gradient after the apply (rescaled);
# measured slower on the headline (2.18 vs 2.09 ms per middle backward pass), off
GRAD_AFTER = os.environ.get("QF_GRAD_AFTER", "0") not in ("0", "", "false")
STREAM_POLY = os.environ.get("QF_STREAM_POLY", "auto")   # auto: R >= 5 (measured: R = 4 keeps the WHT)


def _flit(x: float) -> str:
    return repr(float(np.float32(x))) + "f"


def _sm_idx(c: int) -> str:
    """Shared-memory index tp ^ c of an exchange.  Under planner.swizzle the thread part and the
    register part share only the low nibble (bits >= 4 are distinct local bits), so
    tp ^ c = (tp ^ (c & 15)) + (c & ~15): one XOR per distinct low nibble (common
    subexpression across registers), the rest an immediate LDS/STS offset."""
    lo, hi = c & 15, c & ~15
    if not XADD:
        return f"(tp ^ {c}u)"
    base = f"(tp ^ {lo}u)" if lo else "tp"
    return f"({base} + {hi}u)" if hi else base


def _xor_expr(bits: list, var: str = "t") -> str:
    """XOR over thread bits i of (t bit i ? c_i : 0) with c_i literal."""
    parts = [f"((({var}) >> {i}) & 1u ? {c}u : 0u)" for i, c in enumerate(bits) if c]
    return "(" + " ^ ".join(parts) + ")" if parts else "0u"


def _int_poly(prog, tb: int, te: int):
    """A DIAG op whose angles are all integer multiples m_k of one runtime angle (one symbol,
    one affine map, beta_k = m_k beta_0 -- e.g. a QAOA cost layer): returns (base angle
    column, [m_k], H = sum |m_k|) so the phase exp(-i a0 h) with h = sum_k m_k chi_k is a
    lookup in a per-CTA table of 2H+1 entries; else None."""
    r = prog.recipe
    tsrc = np.asarray(r["term_src"]).reshape(-1, 2)
    tbeta = np.asarray(r["term_beta"])
    cols = [int(prog.term_idx[kk]) for kk in range(tb, te)]
    if not cols:
        return None
    key = None
    for col in cols:
        kind, src = int(tsrc[col][0]), int(tsrc[col][1])
        if kind != 0:
            return None
        k = (int(r["gen_sym"][src]), float(r["gen_coeff"][src]), float(r["gen_const"][src]))
        if key is None:
            key = k
        elif k != key:
            return None
    base = min(cols, key=lambda c: abs(float(tbeta[c])))
    b0 = float(tbeta[base])
    if b0 == 0.0:
        return None
    ms = []
    for col in cols:
        ratio = float(tbeta[col]) / b0
        m = int(round(ratio))
        if m == 0 or abs(ratio - m) > 1e-9:
            return None
        ms.append(m)
    H = sum(abs(m) for m in ms)
    return (base, ms, H) if H <= 255 else None


def _int_grad(prog, tb: int, te: int, ms: list):
    """Gradient weights of an integer-weight phase polynomial: (wb, idm) with every
    non-identity term's weight w_k = wb * m_k, and idm = the identity terms' total multiple
    (their weight is 0: subtracted from h); None when the weights are not of that form."""
    wb, idm = None, 0
    for kk, m in zip(range(tb, te), ms):
        w_ = float(prog.term_w[kk])
        if int(prog.term_mask[kk]) == 0:
            if w_ != 0.0:
                return None
            idm += m
            continue
        if wb is None:
            wb = w_ / m
        elif abs(w_ - wb * m) > 1e-6 * max(1.0, abs(w_)):
            return None
    return (0.0 if wb is None else wb), idm


def _wht_code(vals: dict, R: int, kind: str, out: str, indent: str) -> list:
    """Walsh-Hadamard transform over 2^R entries with symbolic zero tracking.
    vals: S -> variable name (entries absent are zero).  Emits `out{r}` variables."""
    lines = []
    cur = {S: v for S, v in vals.items()}
    tmp_id = [0]
    for j in range(R):
        nxt = {}
        for r in range(1 << R):
            if r & (1 << j):
                continue
            x, y = cur.get(r), cur.get(r | (1 << j))
            if x is None and y is None:
                continue
            a = f"{out}_{j}_{r}"
            b = f"{out}_{j}_{r | (1 << j)}"
            if y is None:
                lines.append(f"{indent}const {kind} {a} = {x}, {b} = {x};")
            elif x is None:
                neg = f"(0u - {y})" if kind == "u32" else f"(-{y})"  # int / float: plain negation
                lines.append(f"{indent}const {kind} {a} = {y}, {b} = {neg};")
            else:
                lines.append(f"{indent}const {kind} {a} = {x} + {y}, {b} = {x} - {y};")
            nxt[r] = a
            nxt[r | (1 << j)] = b
        cur = nxt
    zero = {"u32": "0u", "int": "0"}.get(kind, "0.f")
    for r in range(1 << R):
        lines.append(f"{indent}const {kind} {out}{r} = {cur.get(r, zero)};")
    return lines


def _block_code(D: int, mhi: int, mlo: int, slot_rel: int, gs_store, indent: str, NR: int) -> list:
    """Block-fused adjoint op: after U^dag, the thread's share of the block's two-point matrix
    A = (rho - rho^dag) / 2i, rho[j][k] = sum psi_j conj(lam_k) over the other qubits: D
    diagonal entries, then Re / Im of 2 A[j][k] for j < k (planner.block_slots order).
    Local index bit 1 is register mask ``mhi`` (D = 4), bit 0 ``mlo``."""
    lines = []
    e = 0
    for j in range(D):
        lines.append(indent + gs_store(slot_rel + e, f"blk_entry<{NR}, {mhi}, {mlo}, {j}, {j}, 0>(v0, v1)"))
        e += 1
    for j in range(D):
        for k in range(j + 1, D):
            lines.append(indent + f"{{ const float2 bp = blk_pair<{NR}, {mhi}, {mlo}, {j}, {k}>(v0, v1);")
            lines.append(indent + "  " + gs_store(slot_rel + e, "bp.x"))
            lines.append(indent + "  " + gs_store(slot_rel + e + 1, "bp.y") + " }")
            e += 2
    return lines


def generate(prog: pl.Program, tag: str, remote_pass: int = -1, remote_g: int = 0, fuse: str = None,
             only_pass: int = None, cm: bool = False) -> tuple[list, list, list]:
    """Per-pass CUDA kernel sources (without prelude), kernel names, launch geometry.

    ``remote_pass``: that pass stores into the receive shards of the other ranks instead of
    in place (a global-qubit swap fused into the pass, distributed.py): amplitude ``idx`` of
    rank s goes to rank idx >> (n - g) at (idx & low) | (s << (n - g)).
    ``fuse`` / ``only_pass``: one pass as a part of the turn kernel (``generate_turn``):
    "head" leaves the tile in v0 instead of storing it, "tail" starts from v0 instead of
    loading it.  ``cm``: rotation coefficients from the module's __constant__ slab (CTAU)."""
    n, L, R, adj = prog.n, prog.L, prog.R, prog.adjoint
    TB = L - R
    NR, NT = 1 << R, 1 << TB
    NA = 2 if adj else 1
    # adjoint exchanges psi and lambda one after the other through one tile buffer (half the
    # shared memory per CTA, two more barriers per exchange)
    TILE = 1 << L
    env_minb = int(os.environ.get("QF_MINB_ADJ" if adj else "QF_MINB_FWD", "0"))
    # measured best (tools/sweep.sh): 128 registers for the 12/5 forward (4 CTAs x 128
    # threads), 64 for the 12/4 forward, 128 for the 12/4 adjoint (2 CTAs x 256 threads)
    tuned = {(12, 5, False): 4, (12, 4, False): 4, (12, 4, True): 2, (12, 5, True): 2}.get((L, R, adj))
    minb = env_minb or tuned or max(1, min(8, 65536 // (NT * (NR * 2 * NA + 32))))
    gm = prog.genmats.reshape(-1, 2) if len(prog.genmats) else np.zeros((0, 2), np.float32)
    src = []
    names, geo = [], []
    for pi, p in enumerate(prog.passes):
        if remote_pass >= 0 and pi != remote_pass:
            continue
        if only_pass is not None and pi != only_pass:
            continue
        name = f"qf_{tag}_p{pi}" + ("_rs" if pi == remote_pass else "")
        names.append(name)
        sb, se = int(p[0]), int(p[1])
        init, store = int(p[2]), int(p[3])
        mb, me = int(p[4]), int(p[5])
        ab, ae = int(p[6]), int(p[7])
        slb, sle = int(p[8]), int(p[9])
        n_out = int(p[10])
        cb, ce = int(p[11]), int(p[12])
        outer = [int(x) for x in p[16:16 + n_out]]
        init_mat = [int(x) for x in p[48:48 + n]]
        mcnt, acnt, ccnt, scnt = me - mb, ae - ab, ce - cb, sle - slb
        # merged gradient slots (planner MERGE_SLOTS): register accumulators, stored once at
        # the group's last rotation of the pass
        pass_op_ids = [k for s_ in range(sb, se) for k in range(int(prog.stages[s_][48]),
                                                                 int(prog.stages[s_][49]))]
        merged_last = {}
        for k_ in pass_op_ids:
            if adj and int(prog.ops[k_][14]) and int(prog.ops[k_][7]) >= 0:
                merged_last[int(prog.ops[k_][7])] = k_
        # slot partials: one float per thread and slot, or (many slots) one per warp after a
        # shuffle reduction, so the CTA keeps its occupancy
        n_gate_ops = sum(int(prog.ops[k_][0]) in (pl.OP_DENSE1, pl.OP_DENSE2) for k_ in pass_op_ids)
        # heavy backward passes of the R = 5 rotation programs at 3 CTAs/SM (QF_ADJ3): 168
        # registers, slot partials in a 12-slot ring so that three CTAs' shared memory fits
        adj3 = adj and R == 5 and L == 12 and ADJ3 and not env_minb and not PERSIST and n_gate_ops > SPLIT_LIGHT_OPS
        per_thread_gs = scnt * NT * 4 <= GS_THREAD_BYTES and not (adj3 and scnt > 12)
        # ring of per-thread slots: 32 (flushed as two 16-value chunks under one barrier pair)
        # or 16 (QF_GS_RING)
        RING = 12 if adj3 else GS_RING
        # many slots: a ring of 16 per-thread slots flushed by a 16-value warp transpose-reduction
        # (slots must then be stored in slot order: not with merged accumulators)
        chunked = (not per_thread_gs) and CHUNKED_GS and NT >= 64 and not merged_last
        GSW = NT if (per_thread_gs or chunked) else NT // 32
        ws_floats = (NT // 32) * 32 if (scnt and (per_thread_gs or chunked)) else 0
        gs_slots = min(scnt, RING) if chunked else scnt
        # backward passes of the R = 5 rotation programs with at most SPLIT_LIGHT_OPS gate ops
        # (default: all): psi and lambda exchanged one after the other through one tile buffer,
        # 3 CTAs/SM at 168 registers.  Measured on the headline: turn 1.40 -> 1.29 ms, last pass
        # 1.33 -> 1.31 ms; the 20-op middle passes first spilled (2.07 -> 2.26 ms), and with the
        # immediate-offset exchange addresses (_sm_idx: no spills) gain, 2.07 -> 1.99 ms
        light = (adj and R == 5 and L == 12 and not env_minb and SPLIT_LIGHT_OPS > 0 and not PERSIST
                 and n_gate_ops <= SPLIT_LIGHT_OPS)
        NX = 1 if (adj and (SPLIT_XCHG or light)) else NA
        smem = NX * TILE * 8 + mcnt * 16 + acnt * 4 + ccnt * 4 + gs_slots * GSW * 4 + ws_floats * 4 + 16
        # integer-weight phase polynomials (full-WHT path only) get a per-CTA phase table
        int_tables = {}
        tbl_bytes = 0
        for s_ in range(sb, se):
            stg = prog.stages[s_]
            rg = [int(stg[j]) for j in range(R)]
            for k_ in range(int(stg[48]), int(stg[49])):
                op_ = prog.ops[k_]
                if int(op_[0]) != pl.OP_DIAG:
                    continue
                subs = {pl._bit_subset(int(prog.term_mask[kk]), rg) for kk in range(int(op_[4]), int(op_[5]))}
                kb = {j for S_ in subs for j in range(R) if S_ >> j & 1}
                if (1 << len(kb)) < NR:
                    continue
                ip = _int_poly(prog, int(op_[4]), int(op_[5]))
                if ip is None or ip[0] < ab or ip[0] >= ae:
                    continue
                if adj and int(op_[7]) >= 0 and _int_grad(prog, int(op_[4]), int(op_[5]), ip[1]) is None:
                    continue
                int_tables[k_] = (ip, tbl_bytes)
                tbl_bytes += (2 * ip[2] + 1) * (8 if TB_MODE == "cs" else 16)
        smem = (smem + 15) // 16 * 16 + tbl_bytes
        prefetch = PERSIST_MODE == 2 and init in (pl.INIT_LOAD, pl.INIT_LOAD_PSI)
        NPF = (2 if (adj and init == pl.INIT_LOAD) else 1) if prefetch else 0
        pf_off = smem
        smem += NPF * TILE * 8
        # tensor-core stages (planner tc_blocks): A reuses the exchange tile (16 KB at offset 0,
        # 1024-aligned), then A_lo (16 KB), the B image (8 KB), an mbarrier and the TMEM slot
        tc_stages = [s_ for s_ in range(sb, se) if int(prog.stages[s_][50])] if not adj else []
        if tc_stages:
            assert NT == 128 and NR == 16 and TILE * 8 == 16384, (NT, NR, TILE)
            tc_off = (smem + 1023) // 1024 * 1024
            smem = tc_off + 16384 + 2 * 8192 + 64       # A_lo, two B images (prefetch ring)
        tileq = [q for q in range(n) if q not in set(outer)]

        def dep(l):
            return sum(((l >> i) & 1) << tileq[i] for i in range(L))
        pass_ops = [prog.ops[k] for s_ in range(sb, se) for k in range(int(prog.stages[s_][48]),
                                                                        int(prog.stages[s_][49]))]
        heavy = any(int(op_[0]) == pl.OP_DENSE2 or (int(op_[0]) == pl.OP_DENSE1 and int(op_[9]) == pl.CLS_GENERAL)
                    for op_ in pass_ops)
        minb_p = min(minb, max(1, 65536 // (NT * 128))) if (heavy and not env_minb) else minb
        if light or adj3:
            minb_p = 3
        n_dense2 = sum(int(op_[0]) == pl.OP_DENSE2 for op_ in pass_ops)
        if not adj and R == 5 and n_dense2 >= 4 and not env_minb:
            # 32 amplitudes per thread plus 4x4 matrices spill at 128 registers: 168 (3 CTAs/SM)
            # is faster (QCNN forward passes 21.9 -> 20.3 ms)
            minb_p = min(minb_p, 3)

        # gradient accumulation chains per rotation (R = 5 backward passes at 3 CTAs/SM): 4 in the
        # light passes (turn kernel 1.21 -> 1.17 ms), 1 in the heavy ones (fewer live registers:
        # contiguous middle pass 1.99 -> 1.96 ms), the prelude default (2) elsewhere
        if adj and light and n_gate_ops <= 12:
            chains = int(os.environ.get("QF_GRAD_CHAINS_LIGHT", "4"))
        elif adj and light:
            chains = int(os.environ.get("QF_GRAD_CHAINS_HEAVY", "1"))
        else:
            chains = int(os.environ.get("QF_GRAD_CHAINS", "2"))
        flushes = [0]

        def gs_flush(c0, K):
            """Reduce ring slots [c0, c0+K) (ring position i = slot c0 + i) into partials."""
            NWP = NT // 32
            code = ["{ float x[16];"]
            code += [f"x[{i}] = {f'GS[{i * NT} + t]' if i < K else '0.f'};" for i in range(16)]
            code.append("warp_transpose_sum16(x, t & 31u);")
            if flushes[0]:
                code.append("__syncthreads();")
            code.append("if ((t & 16u) == 0u) WS[(t >> 5) * 32 + (t & 15u)] = x[0];")
            if K > 16:     # second chunk: ring positions 16..K-1 into the upper half of WS
                code += [f"x[{i}] = {f'GS[{(16 + i) * NT} + t]' if 16 + i < K else '0.f'};" for i in range(16)]
                code.append("warp_transpose_sum16(x, t & 31u);")
                code.append("if ((t & 16u) == 0u) WS[(t >> 5) * 32 + 16 + (t & 15u)] = x[0];")
            code.append("__syncthreads();")
            code.append(f"if (t < {K}) {{ double acc = 0.0; for (int wv = 0; wv < {NWP}; ++wv) "
                        f"acc += (double)WS[wv * 32 + t]; a.partials[((size_t)row * a.n_slots + {slb + c0} + t) * "
                        f"{1 << (n - L)} + o] = acc; }}")
            code.append("}")
            flushes[0] += 1
            return " ".join(code)

        def gs_store(slot_rel, expr):
            if per_thread_gs:
                return f"GS[{slot_rel * NT} + t] = {expr};"
            if chunked:
                st = f"GS[{(slot_rel % RING) * NT} + t] = {expr};"
                if slot_rel % RING == RING - 1:
                    st += " " + gs_flush(slot_rel - (RING - 1), RING)
                return st
            return f"{{ const float gsv = warp_sum_f({expr}); if ((t & 31u) == 0u) GS[{slot_rel * GSW} + (t >> 5)] = gsv; }}"
        pad = int(os.environ.get("QF_SMEM_PAD_ADJ" if adj else "QF_SMEM_PAD_FWD", "0"))
        if pad:
            # experiment: dynamic shared memory padded to limit the CTAs per SM (instruction-cache
            # pressure of long straight-line passes vs occupancy)
            smem = max(smem, pad)
        geo.append((NT, smem))
        o = []
        w = o.append
        use_cm = cm and adj and fuse in (None, "tail")
        cm_slots = {}    # staged-slab offset of a rotation coefficient -> its column in qf_cm

        def tau_ref(moff_, pair=False):
            if not use_cm:
                return f"MM[{moff_}].x"
            j = cm_slots.setdefault(moff_, len(cm_slots))
            return f"qf_cm_{tag}[row * @CMK@ + {j}]" + ("" if pair else ".x")
        w(f'extern "C" __global__ void __launch_bounds__({NT}, {minb_p}) {name}(const QfJitArgs a) {{')
        w(f"  extern __shared__ __align__({1024 if tc_stages else 16}) unsigned char smem_raw[];")
        w("  float2* sm = reinterpret_cast<float2*>(smem_raw);")
        # staged matrices: one 16-byte entry {Re, Im, -Im, Im} per element, so a dense apply
        # reads the broadcast real part and the (-Im, Im) pair with one LDS.128
        w(f"  float4* MM = reinterpret_cast<float4*>(sm + {NX * TILE});")
        w(f"  int* ANG = reinterpret_cast<int*>(MM + {mcnt});")
        w(f"  float* CO = reinterpret_cast<float*>(ANG + {acnt});")
        w(f"  float* GS = CO + {ccnt};")
        if ws_floats:
            w(f"  float* WS = GS + {gs_slots * GSW};")
        if int_tables:
            w(f"  {'float2' if TB_MODE == 'cs' else 'float4'}* TB = reinterpret_cast<"
              f"{'float2' if TB_MODE == 'cs' else 'float4'}*>(smem_raw + {(pf_off - tbl_bytes)});")
        if prefetch:
            w(f"  float2* PF = reinterpret_cast<float2*>(smem_raw + {pf_off});")
        w("  const u32 t = threadIdx.x;")
        if tc_stages:
            w(f"  unsigned char* TCAL = smem_raw + {tc_off};")
            w("  unsigned char* TCB = TCAL + 16384;")
            w("  u64* TCM = reinterpret_cast<u64*>(TCB + 16384);")
            w("  u32* TCS = reinterpret_cast<u32*>(TCM + 1);")
            w('  if ((t >> 5) == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;"'
              ' :: "r"(tc_smem(TCS))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }')
            w('  if (t == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(tc_smem(TCM)));'
              ' asm volatile("fence.mbarrier_init.release.cluster;"); }')
            w('  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();'
              ' asm volatile("tcgen05.fence::after_thread_sync;");')
            w("  const u32 tmem = *TCS;")
            w("  u32 tcph = 0u;")
            tc_blocks_here = [int(prog.stages[s_][50]) - 1 for s_ in tc_stages]

            def tc_prefetch(j):
                """cp.async of this pass's j-th tensor-core block's B image into ring slot j % 2."""
                b_ = tc_blocks_here[j]
                return (f"  {{ const float4* __restrict__ tsrc = reinterpret_cast<const float4*>(a.tcb + ((size_t)"
                        f"(blockIdx.x >> {n - L}) * a.tc_n + {b_}) * 2048);"
                        f" for (u32 i = t; i < 512u; i += 128u) {{ const u32 wh = i >> 8, nn = (i >> 3) & 31u, "
                        f"cc = i & 7u; cp_async16(TCB + {(j % 2) * 8192} + wh * 4096u + tc_swz(nn, cc), tsrc + i); }}"
                        f" cp_async_commit(); }}")
            w(tc_prefetch(0))
        for sl in sorted(merged_last):
            w(f"  float gm{sl} = 0.f;")
        if PERSIST:
            # persistent CTAs: a contiguous run of tiles each, so the row's staged matrices,
            # angles and phase tables are rebuilt only when the row changes
            w(f"  const u32 total = (u32)a.pad << {n - L};")
            w("  const u32 per = (total + gridDim.x - 1) / gridDim.x;")
            w("  u32 tile = blockIdx.x * per;")
            w("  const u32 tend = min(total, tile + per);")
            w("  int cur = -1;")
            w(f"  float2 v0[{NR}];")
            if adj:
                w(f"  float2 v1[{NR}];")
            if prefetch:
                # chunk c (16 B = local amplitudes 2c, 2c+1) of thread t: c = t + k * NT
                K = (TILE // 2) // NT
                dt = _xor_expr([dep(2 << i) for i in range(TB)])
                w(f"  const u32 pfd = {dt};")
                w("  auto prefetch = [&](u32 nt) {")
                w(f"    const u32 nrow = nt >> {n - L}, no = nt & {(1 << (n - L)) - 1}u;")
                nb = " | ".join(f"(((no >> {i}) & 1u) << {q})" for i, q in enumerate(outer)) or "0u"
                w(f"    const u32 nbase = {nb};")
                arrays = [("a.psi", 0)] + ([("a.lam", TILE)] if NPF == 2 else [])
                for arr, soff in arrays:
                    w(f"    {{ const float2* __restrict__ src = {arr} + ((size_t)nrow << {n}) + (nbase | pfd);")
                    for k in range(K):
                        w(f"      cp_async16(PF + {soff + 2 * k * NT} + 2 * t, src + {dep(2 * k * NT)}ll);")
                    w("    }")
                w("    cp_async_commit();")
                w("  };")
                w("  if (tile < tend) prefetch(tile);")
            w("  for (; tile < tend; ++tile) {")
            w(f"  const int row = (int)(tile >> {n - L});")
            w(f"  const u32 o = tile & {(1 << (n - L)) - 1}u;")
            w("  if (row != cur) {")
            w("  cur = row;")
            w("  __syncthreads();")
        else:
            w(f"  const int row = (int)(blockIdx.x >> {n - L});")
            w(f"  const u32 o = blockIdx.x & {(1 << (n - L)) - 1}u;")
        mark_stage = len(o)
        if mcnt:
            # stage the row's matrices: as built for the forward sweep; conjugate-transposed
            # (U^dag) for general / X-like / real dense ops of the adjoint sweep
            w(f"  {{ const float2* __restrict__ src = a.mats + (size_t)row * a.n_mat + {mb};")
            w(f"    for (int i = t; i < {mcnt}; i += {NT}) {{ const float2 x = src[i]; MM[i] = make_float4(x.x, x.y, -x.y, x.y); }}")
            if adj:
                # one barrier orders the straight copy before every transposed rewrite (the
                # rewrites of different ops touch disjoint entries)
                first_t = True
                for op_ in pass_ops:
                    kd, cl_ = int(op_[0]), int(op_[9])
                    if kd not in (pl.OP_DENSE1, pl.OP_DENSE2) or cl_ in (pl.CLS_NX, pl.CLS_NY):
                        continue
                    D = 2 if kd == pl.OP_DENSE1 else 4
                    off = int(op_[3]) - mb
                    if first_t:
                        w(f"    __syncthreads();")
                        first_t = False
                    w(f"    if (t < {D * D}) {{ const float2 x = src[{off} + (t % {D}) * {D} + t / {D}];"
                      f" MM[{off} + t] = make_float4(x.x, -x.y, x.y, -x.y); }}")
            w("  }")
        if acnt:
            w(f"  for (int i = t; i < {acnt}; i += {NT}) ANG[i] = a.angles[(size_t)row * a.n_ang + {ab} + i];")
        if ccnt:
            w(f"  for (int i = t; i < {ccnt}; i += {NT}) CO[i] = a.coefs[(size_t)row * a.coef_stride + {cb} + i];")
        if not PERSIST:
            w(f"  float2 v0[{NR}];")
            if adj:
                w(f"  float2 v1[{NR}];")
        w("  __syncthreads();")
        if int_tables:
            for k_, ((bcol, ms, H), off) in int_tables.items():
                ph = f"phase_turns((int)((u32)(h - {H}) * (u32)ANG[{bcol - ab}]), {'true' if adj else 'false'})"
                if TB_MODE == "cs":
                    w(f"  for (int h = t; h < {2 * H + 1}; h += {NT}) TB[{off // 8} + h] = {ph};")
                else:
                    w(f"  for (int h = t; h < {2 * H + 1}; h += {NT}) {{ const float2 ph = {ph};"
                      f" TB[{off // 16} + h] = make_float4(ph.x, ph.x, -ph.y, ph.y); }}")
            w("  __syncthreads();")
        if PERSIST:
            w("  }")
        mark_ptr = len(o)
        base = " | ".join(f"(((o >> {i}) & 1u) << {q})" for i, q in enumerate(outer)) or "0u"
        w(f"  const u32 base = {base};")
        w(f"  float2* __restrict__ psi = a.psi + ((size_t)row << {n});")
        if adj:
            w(f"  float2* __restrict__ lam = a.lam + ((size_t)row << {n});")
        mark_ptr_end = len(o)

        st_rows = [prog.stages[s] for s in range(sb, se)]

        def tglob(st):
            return [1 << int(st[8 + i]) for i in range(TB)]

        def tphys(st):
            return [int(st[32 + i]) for i in range(TB)]

        def roff(st, r, phys=False):
            x = 0
            for j in range(R):
                if r >> j & 1:
                    x ^= int(st[24 + j]) if phys else (1 << int(st[j]))
            return x

        # ---- load / init ----
        mark_load = len(o)
        st0 = st_rows[0]
        w(f"  const u32 gt0 = base | {_xor_expr(tglob(st0))};")
        if fuse == "tail":
            # the turn kernel's backward part: psi is already in registers (the forward part's
            # last stage layout, exchanged to this pass's first stage by generate_turn)
            if adj:
                for r in range(NR):
                    w(f"  v1[{r}] = make_float2(0.f, 0.f);")
        elif prefetch:
            # this tile landed in PF (natural local order) during the previous tile
            def lidx(qs):
                return [1 << tileq.index(q) for q in qs]
            tl = _xor_expr(lidx([int(st0[8 + i]) for i in range(TB)]))
            w("  cp_async_wait_all();")
            w("  __syncthreads();")
            w(f"  {{ const u32 tl0 = {tl};")
            for r in range(NR):
                lo = 0
                for j in range(R):
                    if r >> j & 1:
                        lo |= 1 << tileq.index(int(st0[j]))
                w(f"    v0[{r}] = PF[tl0 ^ {lo}u];")
                if adj:
                    w(f"    v1[{r}] = " + (f"PF[{TILE} + (tl0 ^ {lo}u)];" if NPF == 2 else "make_float2(0.f, 0.f);"))
            w("  }")
            w("  __syncthreads();")
            w("  if (tile + 1 < tend) prefetch(tile + 1);")
        elif init in (pl.INIT_LOAD, pl.INIT_LOAD_PSI):
            # pointer + 64-bit constant offsets: u32 index sums above 2^29 elements were
            # miscompiled (half-width loads) by nvcc/NVRTC 12.9 at n >= 30
            if adj:
                w("  const float2* __restrict__ pt0 = psi + gt0;")
            else:
                w(f"  const float2* __restrict__ pt0 = (a.psi_src ? a.psi_src + ((size_t)row << {n}) : psi) + gt0;")
            if adj and init == pl.INIT_LOAD:
                w("  const float2* __restrict__ lt0 = lam + gt0;")
            vec_ld = int(st0[0]) == 0 and EXP_MODE != "noload"
            for r in range(NR):
                if EXP_MODE == "noload":
                    w(f"  v0[{r}] = make_float2((float)(gt0 + {r}u) * 1e-9f, 0.5f);")
                    if adj:
                        w(f"  v1[{r}] = make_float2(0.25f, (float)(gt0 ^ {r}u) * 1e-9f);")
                    continue
                if vec_ld:
                    # register slot 0 is qubit 0: amplitudes (x, x | 1) in one 16-byte load
                    if r & 1:
                        continue
                    w(f"  ld_pair(pt0 + {roff(st0, r)}ll, v0[{r}], v0[{r + 1}]);")
                    if adj:
                        if init == pl.INIT_LOAD:
                            w(f"  ld_pair(lt0 + {roff(st0, r)}ll, v1[{r}], v1[{r + 1}]);")
                        else:
                            w(f"  v1[{r}] = make_float2(0.f, 0.f); v1[{r + 1}] = make_float2(0.f, 0.f);")
                    continue
                w(f"  v0[{r}] = pt0[{roff(st0, r)}ll];")
                if adj:
                    w(f"  v1[{r}] = " + (f"lt0[{roff(st0, r)}ll];" if init == pl.INIT_LOAD else
                                          "make_float2(0.f, 0.f);"))
        elif init == pl.INIT_ZERO:
            w("  v0[0] = make_float2(gt0 == 0u ? 1.f : 0.f, 0.f);")
            for r in range(1, NR):
                w(f"  v0[{r}] = make_float2(0.f, 0.f);")
        else:
            regq = {int(st0[j]) for j in range(R)}
            w("  float2 c = make_float2(1.f, 0.f);")
            for q in range(n):
                if q in regq:
                    continue
                mo = init_mat[q] if q < len(init_mat) else -1
                if mo < 0:
                    w(f"  if ((gt0 >> {q}) & 1u) c = make_float2(0.f, 0.f);")
                else:
                    w(f"  c = cmul_m(c, MM[((gt0 >> {q}) & 1u) ? {mo - mb + 2} : {mo - mb}]);")
            w("  v0[0] = c;")
            for j in range(R):
                mo = init_mat[int(st0[j])]
                if mo < 0:
                    w(f"  {{ const float2 f0 = make_float2(1.f, 0.f), f1 = make_float2(0.f, 0.f);")
                    for r in range(1 << j):
                        w(f"    v0[{r | (1 << j)}] = cmul(v0[{r}], f1); v0[{r}] = cmul(v0[{r}], f0);")
                else:
                    w(f"  {{ const float4 f0 = MM[{mo - mb}], f1 = MM[{mo - mb + 2}];")
                    for r in range(1 << j):
                        w(f"    v0[{r | (1 << j)}] = cmul_m(v0[{r}], f1); v0[{r}] = cmul_m(v0[{r}], f0);")
                w("  }")

        if (L2PF >= (1 if adj else 2) and not PERSIST and fuse != "tail" and EXP_MODE != "noload"
                and init in (pl.INIT_LOAD, pl.INIT_LOAD_PSI)):
            c_run = 0
            while c_run < L and tileq[c_run] == c_run:
                c_run += 1
            if c_run >= 4:
                runs = 1 << (L - c_run)
                ahead = int(os.environ.get("QF_L2PF_AHEAD", "0")) or minb_p * L2PF_SMS
                nb_ = " | ".join(f"(((no >> {i}) & 1u) << {q})" for i, q in enumerate(outer)) or "0u"
                offx = _xor_expr([1 << tileq[c_run + j] for j in range(L - c_run)], "i") if runs > 1 else "0u"
                srcs_ = ["a.psi"] if adj else ["(a.psi_src ? a.psi_src : a.psi)"]
                if adj and init == pl.INIT_LOAD:
                    srcs_.append("a.lam")
                w(f"  {{ const u32 nb = blockIdx.x + {ahead}u;")
                w("    if (nb < gridDim.x) {")
                w(f"      const u32 nrow = nb >> {n - L}, no = nb & {(1 << (n - L)) - 1}u;")
                w(f"      const u32 nbase = {nb_};")
                w(f"      for (u32 i = t; i < {runs}u; i += {NT}u) {{ const u32 off = nbase | ({offx});")
                for s_ in srcs_:
                    w(f"        l2_prefetch_bulk({s_} + ((size_t)nrow << {n}) + off, {8 << c_run}u);")
                w("      }")
                w("    }")
                w("  }")
        mark_load_end = len(o)
        loads_first = (not adj) or (ADJ_LOADS_FIRST == "1") or (ADJ_LOADS_FIRST == "auto" and n_gate_ops > 12)
        if not PERSIST and not prefetch and loads_first and init in (pl.INIT_LOAD, pl.INIT_LOAD_PSI):
            # backward passes: only the heavy ones (measured on the headline at 3 CTAs/SM: 20-op
            # passes 1.99-2.02 -> 1.95-2.00 ms; the 8/12-op turn and last pass lose 3-5%)
            # issue the tile's global loads before staging the row's matrices / tables, so
            # the staging latency (loads, syncs, table sincos) hides behind the tile loads
            vdecl = [ln for ln in o[mark_stage:mark_ptr] if ln.startswith("  float2 v0[") or
                     ln.startswith("  float2 v1[")]
            staging = [ln for ln in o[mark_stage:mark_ptr] if ln not in vdecl]
            o[mark_stage:mark_load_end] = (vdecl + o[mark_ptr:mark_ptr_end] + o[mark_load:mark_load_end] + staging)
        # ---- stages ----
        for si, st in enumerate(st_rows if EXP_MODE != "memonly" else []):
            if si:
                prev = st_rows[si - 1]
                if PERSIST or (si > 1 and (PREW_SYNC or tc_stages)):
                    # readers of the previous exchange must be done before it is overwritten.
                    # Without it: a thread writes exactly the addresses it read itself in the
                    # previous exchange (both in layout `prev`), so there is no cross-thread
                    # hazard; the first exchange of a tile has no earlier readers at all
                    w("  __syncthreads();")
                if NX == 1 and adj:
                    for vv in ("v0", "v1"):
                        if vv == "v1":
                            w("  __syncthreads();")
                        w(f"  {{ const u32 tp = {_xor_expr(tphys(prev))};")
                        for r in range(NR):
                            w(f"    sm[{_sm_idx(roff(prev, r, True))}] = {vv}[{r}];")
                        w("  }")
                        w("  __syncthreads();")
                        w(f"  {{ const u32 tp = {_xor_expr(tphys(st))};")
                        for r in range(NR):
                            w(f"    {vv}[{r}] = sm[{_sm_idx(roff(st, r, True))}];")
                        w("  }")
                else:
                    w(f"  {{ const u32 tp = {_xor_expr(tphys(prev))};")
                    for r in range(NR):
                        w(f"    sm[{_sm_idx(roff(prev, r, True))}] = v0[{r}];")
                        if adj:
                            w(f"    sm[{TILE} + {_sm_idx(roff(prev, r, True))}] = v1[{r}];")
                    w("  }")
                    w("  __syncthreads();")
                    w(f"  {{ const u32 tp = {_xor_expr(tphys(st))};")
                    for r in range(NR):
                        w(f"    v0[{r}] = sm[{_sm_idx(roff(st, r, True))}];")
                        if adj:
                            w(f"    v1[{r}] = sm[{TILE} + {_sm_idx(roff(st, r, True))}];")
                    w("  }")
            reg_glob = [int(st[j]) for j in range(R)]
            need_gt = any(int(prog.ops[k][0]) in (pl.OP_DIAG, pl.OP_OBS) for k in range(int(st[48]), int(st[49])))
            if need_gt:
                w(f"  {{ const u32 gt = base | {_xor_expr(tglob(st))};")
            else:
                w("  {")
            if int(st[50]) and not adj:
                blk = int(st[50]) - 1
                j_tc = tc_stages.index(sb + si)
                w(f"    // tensor-core stage: the product of this stage's {int(st[49]) - int(st[48])} dense ops, "
                  f"one 16 x 16 unitary (tc block {blk}); its B image was prefetched into ring slot {j_tc % 2}")
                w("    cp_async_wait_all();")
                w("    __syncthreads();   // B landed for every thread; the exchange's reads of the tile are done")
                if j_tc + 1 < len(tc_stages):
                    w("  " + tc_prefetch(j_tc + 1))
                w("    #pragma unroll")
                w("    for (u32 c = 0; c < 8u; ++c) {")
                w("      const float4 x = make_float4(v0[2 * c].x, v0[2 * c].y, v0[2 * c + 1].x, v0[2 * c + 1].y);")
                w("      const float4 lo = make_float4(tf32_lo(x.x), tf32_lo(x.y), tf32_lo(x.z), tf32_lo(x.w));")
                w("      // explicit tf32 hi part: the MMA's own fp32 -> tf32 conversion may round, and the")
                w("      // split must satisfy hi + lo == x exactly")
                w("      *reinterpret_cast<float4*>(smem_raw + tc_swz(t, c)) = make_float4(x.x - lo.x, x.y - lo.y, "
                  "x.z - lo.z, x.w - lo.w);")
                w("      *reinterpret_cast<float4*>(TCAL + tc_swz(t, c)) = lo;")
                w("    }")
                w('    asm volatile("fence.proxy.async.shared::cta;"); asm volatile("tcgen05.fence::before_thread_sync;");')
                w('    __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");')
                w(f"    if (t == 0) tc_block_mma(tmem, smem_raw, TCAL, TCB + {(j_tc % 2) * 8192}, TCM);")
                w("    tc_wait(TCM, tcph); tcph ^= 1u;")
                w('    asm volatile("tcgen05.fence::after_thread_sync;");')
                w("    tc_ld(tmem + (((t >> 5) * 32u) << 16), v0);")
                w('    asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();'
                  ' asm volatile("tcgen05.fence::after_thread_sync;");')
            for k in (range(int(st[48]), int(st[49])) if (EXP_MODE != "nocompute" and not (int(st[50]) and not adj))
                      else []):
                op = prog.ops[k]
                kind = int(op[0])
                if EXP_MODE == "nodiag" and kind == pl.OP_DIAG:
                    continue
                s0, s1, moff = int(op[1]), int(op[2]), int(op[3]) - mb
                slot = int(op[7])
                cls, gk = int(op[9]), int(op[10])
                if kind == pl.OP_DENSE1 and int(op[15]):
                    # lane op: normalised X rotation on thread bit op[15] - 1 (warp shuffles)
                    assert cls == pl.CLS_NX and int(op[15]) <= 5, (cls, int(op[15]))
                    m = 1 << (int(op[15]) - 1)
                    w(f"    {{ const float tau = {tau_ref(moff)};")
                    if adj and slot >= 0:
                        assert gk == pl.GK_X and not int(op[14])
                        sc = float(gm[int(op[8]) + 4, 0])
                        w("      " + gs_store(slot - slb, f"{_flit(sc)} * laneGradNX<{NR}>(v0, v1, tau, {m}u)") + " }")
                    elif adj:
                        w(f"      laneNX2<{NR}>(v0, v1, tau, {m}u); }}")
                    else:
                        w(f"      laneNX<{NR}>(v0, tau, {m}u); }}")
                    continue
                if kind == pl.OP_DENSE1 and cls in (pl.CLS_NX, pl.CLS_NY):
                    # Pauli-frame normalised rotation: the build step wrote tau (adjoint-ready)
                    ax = 1 if cls == pl.CLS_NX else 2
                    if use_cm and adj and not FUSED_GRAD and not GRAD_AFTER and not int(op[14]):
                        # (tau, tau) pair from the constant slab: one LDCU.64, no pair building
                        w(f"    {{ const float2 tau = {tau_ref(moff, pair=True)};")
                    else:
                        w(f"    {{ const float tau = {tau_ref(moff)};")
                    if adj and slot >= 0 and FUSED_GRAD and not int(op[14]):
                        g0 = int(op[8])
                        sc = float(gm[g0 + 4, 0])
                        w("      " + gs_store(slot - slb, f"{_flit(sc)} * gradApplyN<{s0}, {NR}, {gk}, {ax}>(v0, v1, tau)"))
                        w("    }")
                        continue
                    if adj and slot >= 0 and int(op[14]):
                        # merged slot: weight = this rotation's frame scale relative to the head
                        g0 = int(op[8])
                        sc = float(gm[g0 + 4, 0])
                        w(f"      gm{slot} = fmaf(MM[{moff}].y, {_flit(sc)} * gradp<{s0}, {NR}, {gk}>(v0, v1), gm{slot});")
                        if merged_last[slot] == k:
                            w("      " + gs_store(slot - slb, f"gm{slot}"))
                    elif adj and slot >= 0 and GRAD_AFTER:
                        # gradient AFTER the apply: M = I - i tau Q commutes with Q and M^dag M =
                        # (1 + tau^2) I, so <M lam|Q|M psi> = (1 + tau^2) <lam|Q|psi>.  The
                        # gradient's accumulation chains then overlap the next rotation's applies
                        # (both only read the new values) instead of delaying them
                        g0 = int(op[8])
                        sc = float(gm[g0 + 4, 0])
                        w(f"      applyN<{s0}, {NR}, {ax}>(v1, tau);")
                        w(f"      applyN<{s0}, {NR}, {ax}>(v0, tau);")
                        w("      " + gs_store(slot - slb, f"__fdividef({_flit(sc)}, fmaf(tau, tau, 1.f)) * "
                                                          f"gradp<{s0}, {NR}, {gk}>(v0, v1)") + " }")
                        continue
                    elif adj and slot >= 0:
                        g0 = int(op[8])
                        sc = float(gm[g0 + 4, 0])
                        w("      " + gs_store(slot - slb, f"{_flit(sc)} * gradp<{s0}, {NR}, {gk}, {chains}>(v0, v1)"))
                    if adj:
                        w(f"      applyN<{s0}, {NR}, {ax}>(v1, tau);")
                    w(f"      applyN<{s0}, {NR}, {ax}>(v0, tau); }}")
                elif kind == pl.OP_DENSE1:
                    # adjoint: apply U^dag first, then the gradient slot -- G commutes with
                    # U = exp(-i v G), so Im<lam|G|psi> is the same on either side, and after
                    # the apply the Pauli frame on the op's qubits has been absorbed
                    w(f"    {{ const float2 u00 = mm2(MM, {moff}), u01 = mm2(MM, {moff + 1}), u10 = mm2(MM, {moff + 2}),"
                      f" u11 = mm2(MM, {moff + 3});")
                    if cls == pl.CLS_GENERAL:
                        if adj:
                            w(f"      apply1m<{s0}, {NR}>(v1, MM + {moff});")
                        w(f"      apply1m<{s0}, {NR}>(v0, MM + {moff});")
                    else:
                        if adj:
                            w(f"      apply1<{s0}, {NR}, {cls}>(v1, u00, u01, u10, u11);")
                        w(f"      apply1<{s0}, {NR}, {cls}>(v0, u00, u01, u10, u11);")
                    if adj and slot >= 0 and int(op[13]):
                        o.extend(_block_code(2, 0, 1 << s0, slot - slb, gs_store, "      ", NR))
                    elif adj and slot >= 0:
                        g0 = int(op[8])
                        if gk:
                            sc = float(gm[g0 + 4, 0])
                            w(f"      const float gacc = {_flit(sc)} * gradp<{s0}, {NR}, {gk}>(v0, v1);")
                        else:
                            gl = [f"make_float2({_flit(gm[g0 + i, 0])}, {_flit(gm[g0 + i, 1])})" for i in range(4)]
                            w(f"      const float gacc = grad1<{s0}, {NR}>(v0, v1, {', '.join(gl)});")
                        w("      " + gs_store(slot - slb, "gacc"))
                    w("    }")
                elif kind == pl.OP_DENSE2 and cls == pl.CLS_NP:
                    code = int(op[12])
                    w(f"    {{ const float tau = {tau_ref(moff)};")
                    if adj and slot >= 0:
                        g0 = int(op[8])
                        sc = float(gm[g0 + 16, 0])
                        w("      " + gs_store(slot - slb, f"{_flit(sc)} * gradNP<{s0}, {s1}, {NR}, {code}>(v0, v1)"))
                    if adj:
                        w(f"      applyNP<{s0}, {s1}, {NR}, {code}>(v1, tau);")
                    w(f"      applyNP<{s0}, {s1}, {NR}, {code}>(v0, tau); }}")
                elif kind == pl.OP_DENSE2:
                    if adj:
                        w("    {")
                        w(f"      apply2m<{s0}, {s1}, {NR}>(v0, MM + {moff});"
                          f" apply2m<{s0}, {s1}, {NR}>(v1, MM + {moff});")
                        if slot >= 0 and int(op[13]):
                            o.extend(_block_code(4, 1 << s0, 1 << s1, slot - slb, gs_store, "      ", NR))
                        elif slot >= 0:
                            g0 = int(op[8])
                            gl = ", ".join(f"make_float2({_flit(gm[g0 + i, 0])}, {_flit(gm[g0 + i, 1])})"
                                           for i in range(16))
                            w(f"      const float2 g[16] = {{{gl}}};")
                            w("      " + gs_store(slot - slb, f"grad2<{s0}, {s1}, {NR}>(v0, v1, g)"))
                        w("    }")
                    else:
                        w(f"    apply2m<{s0}, {s1}, {NR}>(v0, MM + {moff});")
                elif kind in (pl.OP_DIAG, pl.OP_OBS):
                    tb, te = int(op[4]), int(op[5])
                    groups: dict = {}
                    for kk in range(tb, te):
                        S = pl._bit_subset(int(prog.term_mask[kk]), reg_glob)
                        groups.setdefault(S, []).append(kk)
                    pre = f"d{k}"
                    w("    {")
                    xcol = int(op[11])
                    gv = "gt"
                    if xcol >= 0:   # Pauli frame: evaluate at index ^ x
                        gv = f"{pre}gx"
                        w(f"      const u32 {gv} = gt ^ (u32)ANG[{xcol - ab}];")
                    # register slots the phase polynomial depends on: with 2^k < 2^R distinct
                    # values per thread, evaluate 2^k phases (table) instead of one per amplitude
                    kbits = sorted({j for S in groups for j in range(R) if S >> j & 1})
                    table = (1 << len(kbits)) < NR

                    def cidx(r):
                        return sum(((r >> j) & 1) << i for i, j in enumerate(kbits))

                    def csub(S):
                        return sum(((S >> j) & 1) << i for i, j in enumerate(kbits))

                    def signed_sum(names_by_S, c, zero):
                        parts = []
                        for S, nm in names_by_S.items():
                            neg = bin(csub(S) & c).count("1") & 1
                            parts.append(("-" if neg else "+") + nm)
                        if not parts:
                            return zero
                        e = " ".join(parts)
                        return e[1:] if e[0] == "+" else "(" + zero + " " + e + ")"

                    if kind == pl.OP_DIAG and k in int_tables:
                        (bcol, ms, H), off = int_tables[k]
                        kks = list(range(tb, te))
                        # h_S = sum_k m_k (-1)^{popc(gx & mask_k)}.  Every term of group S has the
                        # same register bits (S), whose parity in gx (the Pauli-frame x mask there:
                        # gt is 0 on register bits) is one sign for the group; the bits outside the
                        # registers are counted in bulk: sum_k m (1 - 2 bit) = m (K - 2 popc(gx & M))
                        # for single bits, and with y_d = gx ^ (gx >> d) for pairs at distance d
                        regmask = sum(1 << q for q in reg_glob)
                        ydist = {}
                        hexpr = {}
                        for S, ks in groups.items():
                            const = 0
                            bulk: dict = {}
                            rest = []
                            for kk in ks:
                                om = int(prog.term_mask[kk]) & ~regmask
                                mk = ms[kks.index(kk)]
                                bits = [b for b in range(32) if om >> b & 1]
                                if len(bits) == 0:
                                    const += mk
                                elif len(bits) == 1:
                                    key = ("s", 0, mk)
                                    bulk.setdefault(key, [0, 0])
                                    bulk[key][0] |= 1 << bits[0]
                                    bulk[key][1] += 1
                                elif len(bits) == 2:
                                    d = bits[1] - bits[0]
                                    key = ("p", d, mk)
                                    bulk.setdefault(key, [0, 0])
                                    bulk[key][0] |= 1 << bits[0]
                                    bulk[key][1] += 1
                                    ydist[d] = True
                                else:
                                    rest.append((om, mk))
                            parts = [str(const)] if const else []
                            for (typ, d, mk), (msk, cnt) in bulk.items():
                                srcv = gv if typ == "s" else f"{pre}y{d}"
                                parts.append(f"{mk} * ({cnt} - 2 * __popc({srcv} & {msk}u))")
                            for om, mk in rest:
                                parts.append(f"((__popc({gv} & {om}u) & 1) ? {-mk} : {mk})")
                            hexpr[S] = " + ".join(parts) or "0"
                        for d in sorted(ydist):
                            w(f"      const u32 {pre}y{d} = {gv} ^ ({gv} >> {d});")
                        for S in groups:
                            rsm = sum(1 << reg_glob[j] for j in range(R) if S >> j & 1)
                            if rsm and xcol >= 0:   # frame x bits on the group's register qubits
                                w(f"      const int {pre}h{S} = ((__popc({gv} & {rsm}u) & 1) ? -1 : 1) * ({hexpr[S]});")
                            else:
                                w(f"      const int {pre}h{S} = {hexpr[S]};")
                        if (R >= 5 if STREAM_POLY == "auto" else STREAM_POLY not in ("0", "", "false")):
                            # streaming evaluation in Gray-code order: one live h value instead
                            # of 2^R (register pressure), each step adds the flipped bit's terms
                            grad_here = adj and slot >= 0
                            NQ = 4 if NR >= 16 else 1      # independent gradient chains (ILP)
                            if grad_here:
                                wb, idm = _int_grad(prog, tb, te, ms)
                                w("      " + " ".join(f"float gq{c} = 0.f;" for c in range(NQ)))
                            for S in groups:
                                if S:
                                    w(f"      const int {pre}t{S} = 2 * {pre}h{S};")
                            w(f"      int {pre}Hc = {' + '.join(f'{pre}h{S}' for S in groups) or '0'};")
                            prev = 0
                            for i in range(NR):
                                r = i ^ (i >> 1)
                                if i:
                                    j = (r ^ prev).bit_length() - 1
                                    parts = []
                                    for S in groups:
                                        if S >> j & 1:
                                            neg = bin(S & prev).count("1") & 1   # current sign of h_S
                                            parts.append(("+" if neg else "-") + f"{pre}t{S}")
                                    if parts:
                                        w(f"      {pre}Hc = {pre}Hc {' '.join(parts)};")
                                prev = r
                                if grad_here:
                                    hr = f"{pre}Hc" if not idm else f"({pre}Hc - {idm})"
                                    c = i % NQ
                                    w(f"      gq{c} = fmaf((float){hr}, im_conj_mul(v1[{r}], v0[{r}]), gq{c});")
                                if TB_MODE == "cs":
                                    w(f"      {{ const float2 T = TB[{off // 8 + H} + {pre}Hc];"
                                      f" v0[{r}] = cmul_cs(v0[{r}], T);" +
                                      (f" v1[{r}] = cmul_cs(v1[{r}], T);" if adj else "") + " }")
                                else:
                                    w(f"      {{ const float4 T = TB[{off // 16 + H} + {pre}Hc];"
                                      f" const u64 P = pk(T.x, T.y), N = pk(T.z, T.w);"
                                      f" v0[{r}] = upk(f2fma(N, pk(v0[{r}].y, v0[{r}].x), f2mul(P, pk(v0[{r}].x, v0[{r}].y))));" +
                                      (f" v1[{r}] = upk(f2fma(N, pk(v1[{r}].y, v1[{r}].x), f2mul(P, pk(v1[{r}].x, v1[{r}].y))));"
                                       if adj else "") + " }")
                            if grad_here:
                                tot = " + ".join(f"gq{c}" for c in range(NQ))
                                w("      " + gs_store(slot - slb, f"{_flit(wb)} * ({tot})"))
                            continue_stream = True
                        else:
                            continue_stream = False
                        if not continue_stream:
                          o.extend(_wht_code({S: f"{pre}h{S}" for S in groups}, R, "int", f"{pre}H", "      "))
                        if adj and slot >= 0 and not continue_stream:
                            wb, idm = _int_grad(prog, tb, te, ms)
                            w("      float gq = 0.f;")
                            for r in range(NR):
                                hr = f"{pre}H{r}" if not idm else f"({pre}H{r} - {idm})"
                                w(f"      gq = fmaf((float){hr}, im_conj_mul(v1[{r}], v0[{r}]), gq);")
                            w("      " + gs_store(slot - slb, f"{_flit(wb)} * gq"))
                        for r in (range(NR) if not continue_stream else []):
                            if TB_MODE == "cs":
                                w(f"      {{ const float2 T = TB[{off // 8 + H} + {pre}H{r}];"
                                  f" v0[{r}] = cmul_cs(v0[{r}], T);" +
                                  (f" v1[{r}] = cmul_cs(v1[{r}], T);" if adj else "") + " }")
                            else:
                                w(f"      {{ const float4 T = TB[{off // 16 + H} + {pre}H{r}];"
                                  f" const u64 P = pk(T.x, T.y), N = pk(T.z, T.w);"
                                  f" v0[{r}] = upk(f2fma(N, pk(v0[{r}].y, v0[{r}].x), f2mul(P, pk(v0[{r}].x, v0[{r}].y))));" +
                                  (f" v1[{r}] = upk(f2fma(N, pk(v1[{r}].y, v1[{r}].x), f2mul(P, pk(v1[{r}].x, v1[{r}].y))));"
                                   if adj else "") + " }")
                    elif kind == pl.OP_DIAG:
                        if adj and slot >= 0:
                            bnames = {}
                            for S, ks in groups.items():
                                acc = f"{pre}b{S}"
                                w(f"      float {acc} = 0.f;")
                                for kk in ks:
                                    wt = float(prog.term_w[kk])
                                    if wt == 0.0:
                                        continue
                                    m = int(prog.term_mask[kk])
                                    w(f"      {acc} += (__popc({gv} & {m}u) & 1) ? {_flit(-wt)} : {_flit(wt)};")
                                bnames[S] = acc
                            if table:
                                # grad = sum_c h[c] * sum_{r: c(r)=c} Im(conj(lam_r) psi_r)
                                terms_acc = []
                                for c in range(1 << len(kbits)):
                                    rs = [r for r in range(NR) if cidx(r) == c]
                                    w(f"      float {pre}q{c} = 0.f;")
                                    for r in rs:
                                        w(f"      {pre}q{c} = fmaf(v1[{r}].x, v0[{r}].y, fmaf(-v1[{r}].y, v0[{r}].x, {pre}q{c}));")
                                    terms_acc.append(f"({signed_sum(bnames, c, '0.f')}) * {pre}q{c}")
                                w("      " + gs_store(slot - slb, " + ".join(terms_acc) or "0.f"))
                            else:
                                # gradient: sum_S W[S] * B[S], W = WHT(Im(conj(lam) psi)), B[S] = sum w_k sign_k
                                for r in range(NR):
                                    w(f"      const float {pre}w{r} = im_conj_mul(v1[{r}], v0[{r}]);")
                                wl = _wht_code({r: f"{pre}w{r}" for r in range(NR)}, R, "float", f"{pre}W", "      ")
                                o.extend(wl)
                                terms_acc = [f"{pre}W{S} * {bnames[S]}" for S in bnames]
                                w("      " + gs_store(slot - slb, " + ".join(terms_acc) or "0.f"))
                        for S, ks in groups.items():
                            w(f"      u32 {pre}a{S} = 0u;")
                            for kk in ks:
                                m = int(prog.term_mask[kk])
                                col = int(prog.term_idx[kk]) - ab
                                w(f"      {{ const u32 x = (u32)ANG[{col}]; {pre}a{S} += (__popc({gv} & {m}u) & 1) ? (0u - x) : x; }}")
                        inv = 'true' if adj else 'false'
                        if table:
                            anames = {S: f"{pre}a{S}" for S in groups}
                            for c in range(1 << len(kbits)):
                                w(f"      const float2 {pre}P{c} = phase_turns((int)({signed_sum(anames, c, '0u')}), {inv});")
                                w(f"      const u64 {pre}N{c} = pk_negpos({pre}P{c}.y);")
                            for r in range(NR):
                                c = cidx(r)
                                w(f"      v0[{r}] = cmulp(v0[{r}], {pre}P{c}.x, {pre}N{c});" +
                                  (f" v1[{r}] = cmulp(v1[{r}], {pre}P{c}.x, {pre}N{c});" if adj else ""))
                        else:
                            o.extend(_wht_code({S: f"{pre}a{S}" for S in groups}, R, "u32", f"{pre}A", "      "))
                            for r in range(NR):
                                w(f"      {{ const float2 ph = phase_turns((int){pre}A{r}, {inv});"
                                  f" v0[{r}] = cmul(v0[{r}], ph);" + (f" v1[{r}] = cmul(v1[{r}], ph);" if adj else "") + " }")
                    else:  # OBS
                        for S, ks in groups.items():
                            w(f"      float {pre}a{S} = 0.f;")
                            for kk in ks:
                                m = int(prog.term_mask[kk])
                                col = -1 - int(prog.term_idx[kk]) - cb
                                w(f"      {{ const float x = CO[{col}]; {pre}a{S} += (__popc({gv} & {m}u) & 1) ? -x : x; }}")
                        if table:
                            anames = {S: f"{pre}a{S}" for S in groups}
                            for c in range(1 << len(kbits)):
                                w(f"      const float {pre}C{c} = {signed_sum(anames, c, '0.f')};")
                            coef = {r: f"{pre}C{cidx(r)}" for r in range(NR)}
                        else:
                            o.extend(_wht_code({S: f"{pre}a{S}" for S in groups}, R, "float", f"{pre}A", "      "))
                            coef = {r: f"{pre}A{r}" for r in range(NR)}
                        w("      float e = 0.f;")
                        for r in range(NR):
                            w(f"      e = fmaf({coef[r]}, fmaf(v0[{r}].x, v0[{r}].x, v0[{r}].y * v0[{r}].y), e);")
                            if adj:
                                w(f"      v1[{r}] = cscale({coef[r]}, v0[{r}]);")
                        if slot >= 0:
                            w("      " + gs_store(slot - slb, "e"))
                    w("    }")
            w("  }")

        # ---- store ----
        if store and fuse != "head":
            stl = st_rows[-1]
            if int(p[126]):
                # relabelled pass (planner.plan_passes_remap): tile bit at physical position
                # tileq[i] is stored to physical position p[84 + i]
                out_of = {tileq[i]: int(p[84 + i]) for i in range(L)}
                stl = stl.copy()
                for j in range(R):
                    stl[j] = out_of[int(stl[j])]
                for i in range(TB):
                    stl[8 + i] = out_of[int(stl[8 + i])]
            w(f"  {{ const u32 gs = base | {_xor_expr(tglob(stl))};")
            if pi == remote_pass:
                SH = n - remote_g
                low = (1 << SH) - 1
                w("    const u32 myr = (u32)(a.rank_base + row);")
                for r in range(NR):
                    w(f"    {{ const u32 idx = gs + {roff(stl, r)}u;"
                      f" a.peers[idx >> {SH}][(size_t)((idx & {low}u) | (myr << {SH}))] = v0[{r}]; }}")
            else:
                w("    float2* __restrict__ pts = psi + gs;")
            if adj and pi != remote_pass:
                w("    float2* __restrict__ lts = lam + gs;")
            # register slot 0 is qubit 0: amplitudes (x, x | 1) in one 16-byte store
            vec_st = int(stl[0]) == 0 and not int(p[126])

            def st_all(ptr, v, ind):
                for r in range(NR):
                    if vec_st:
                        if not r & 1:
                            w(f"{ind}st_pair({ptr} + {roff(stl, r)}ll, {v}[{r}], {v}[{r + 1}]);")
                    else:
                        w(f"{ind}{ptr}[{roff(stl, r)}ll] = {v}[{r}];")
            if adj and pi != remote_pass:
                w("    if (!a.skip_psi) {")
                st_all("pts", "v0", "      ")
                w("    }")
                st_all("lts", "v1", "    ")
            if pi != remote_pass and not adj:
                st_all("pts", "v0", "    ")
            w("  }")
        if scnt and chunked:
            if scnt % RING:
                w("  " + gs_flush(scnt - scnt % RING, scnt % RING))
        elif scnt and per_thread_gs and NT >= 64:
            # each thread's slot values are its own GS entries: per 32-slot chunk, a warp
            # transpose-reduction leaves slot L's warp sum on lane L; warps combine in order
            NWP = NT // 32
            for c0 in range(0, scnt, 32):
                K = min(32, scnt - c0)
                w("  {")
                w("    float x[32];")
                for i in range(32):
                    w(f"    x[{i}] = {f'GS[{(c0 + i) * NT} + t]' if i < K else '0.f'};")
                w("    warp_transpose_sum32(x, t & 31u);")
                if c0 or PERSIST:
                    w("    __syncthreads();")   # the previous chunk's cross-warp reads are done
                w(f"    WS[(t >> 5) * 32 + (t & 31)] = x[0];")
                w("    __syncthreads();")
                w(f"    if (t < {K}) {{ double acc = 0.0;")
                w(f"      for (int wv = 0; wv < {NWP}; ++wv) acc += (double)WS[wv * 32 + t];")
                w(f"      a.partials[((size_t)row * a.n_slots + {slb + c0} + t) * {1 << (n - L)} + o] = acc; }}")
                w("  }")
        elif scnt:
            w("  __syncthreads();")
            w(f"  for (int s = t >> 5; s < {scnt}; s += {max(NT // 32, 1)}) {{")
            w("    double acc = 0.0;")
            w(f"    for (int i = (t & 31); i < {GSW}; i += 32) acc += (double)GS[s * {GSW} + i];")
            w("    acc = warp_sum_d(acc);")
            w(f"    if ((t & 31) == 0) a.partials[((size_t)row * a.n_slots + {slb} + s) * {1 << (n - L)} + o] = acc;")
            w("  }")
        if PERSIST:
            if scnt:
                w("  __syncthreads();   // slot partials are rewritten by the next tile")
            w("  }")
        if tc_stages:
            w('  if ((t >> 5) == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" :: "r"(tmem));')
        w("}")
        code = "\n".join(o) + "\n"
        if cm_slots:
            # the slab's columns: the pass's slab offsets (relative to its first matrix) in
            # column order; JitProgram gathers them per row into the module's constant array
            cols = ",".join(str(mb + m_) for m_ in cm_slots)
            code = (f"// QF_CM_COLS {cols}\n__constant__ float2 qf_cm_{tag}[{CM_CAP}];\n" +
                    code.replace("@CMK@", str(len(cm_slots))))
        src.append(code)
    return src, names, geo


def _turn_compatible(fwd: pl.Program, adj: pl.Program) -> bool:
    """The turn kernel joins the forward's last pass and the backward's first pass: both
    programs must be checkpoint mirrors with the same tile geometry."""
    if not (adj.adjoint and not fwd.adjoint and fwd.L == adj.L and fwd.R == adj.R and fwd.n == adj.n):
        return False
    P = len(fwd.passes)
    if P != len(adj.passes) or P < 2:
        return False
    pf, pa = fwd.passes[P - 1], adj.passes[0]
    outer_f = sorted(int(x) for x in pf[16:16 + int(pf[10])])
    outer_a = sorted(int(x) for x in pa[16:16 + int(pa[10])])
    return outer_f == outer_a and int(pa[2]) == pl.INIT_LOAD_PSI and not int(pf[126])


def generate_turn(fwd: pl.Program, adj: pl.Program, name: str = "qf_turn", cm: bool = False) -> tuple[str, int, int]:
    """One kernel for the forward's last tile pass and the backward's first (checkpointed,
    lambda = H psi fused): the final state never leaves registers -- no store of it by the
    forward, no load of it by the backward.  Parameters (forward args ``a``, backward args
    ``b``).  Returns (source, threads per CTA, dynamic smem bytes)."""
    P = len(fwd.passes)
    fs, _, fg = generate(fwd, "f", fuse="head", only_pass=P - 1)
    bs, _, bg = generate(adj, "a", fuse="tail", only_pass=0, cm=cm)
    prefix = ""
    if bs[0].startswith("// QF_CM_COLS "):       # the backward half's constant slab
        head, decl, rest = bs[0].split("\n", 2)
        prefix, bs = head + "\n" + decl + "\n", [rest]
    NT, NR = fg[0][0], 1 << fwd.R
    assert bg[0][0] == NT
    import re

    def body(src):
        lines = src.rstrip("\n").split("\n")
        head = lines[0]
        m = re.search(r"__launch_bounds__\((\d+), (\d+)\)", head)
        keep = [ln for ln in lines[1:-1] if ln not in (
            "  extern __shared__ __align__(16) unsigned char smem_raw[];",
            f"  float2 v0[{NR}];", f"  float2 v1[{NR}];")]
        return keep, int(m.group(2))

    fb, mf = body(fs[0])
    ab, ma = body(bs[0])
    ab = [re.sub(r"\ba\.", "b.", ln) for ln in ab]
    o = [f'extern "C" __global__ void __launch_bounds__({NT}, {min(mf, ma)}) {name}(const QfJitArgs a, '
         f'const QfJitArgs b) {{',
         "  extern __shared__ __align__(16) unsigned char smem_raw[];",
         f"  float2 v0[{NR}];", f"  float2 v1[{NR}];", "  {"] + fb + ["  }", "  __syncthreads();"]
    # forward's last stage layout -> backward's first stage layout (if they differ)
    R, TB = fwd.R, fwd.L - fwd.R
    sf = fwd.stages[int(fwd.passes[P - 1][1]) - 1]
    sa = adj.stages[int(adj.passes[0][0])]
    same = all(int(sf[j]) == int(sa[j]) for j in range(R)) and all(int(sf[8 + i]) == int(sa[8 + i]) for i in range(TB))
    if not same:
        def tp(st):
            return _xor_expr([int(st[32 + i]) for i in range(TB)])

        def ro(st, r):
            x = 0
            for j in range(R):
                if r >> j & 1:
                    x ^= int(st[24 + j])
            return x
        o.append("  { float2* sm = reinterpret_cast<float2*>(smem_raw); const u32 t = threadIdx.x;")
        o.append(f"    {{ const u32 tp = {tp(sf)};")
        o += [f"      sm[{_sm_idx(ro(sf, r))}] = v0[{r}];" for r in range(NR)]
        o.append("    }")
        o.append("    __syncthreads();")
        o.append(f"    {{ const u32 tp = {tp(sa)};")
        o += [f"      v0[{r}] = sm[{_sm_idx(ro(sa, r))}];" for r in range(NR)]
        o.append("    }")
        o.append("    __syncthreads();")
        o.append("  }")
    o += ["  {"] + ab + ["  }", "}"]
    return prefix + "\n".join(o) + "\n", NT, max(fg[0][1], bg[0][1])


class QfTurnArgs(C.Structure):
    _fields_ = [("a", QfJitArgs), ("b", QfJitArgs)]


class TurnKernel:
    """The compiled turn kernel of one (forward, backward) program pair."""

    def __init__(self, fwd: pl.Program, adj: pl.Program, device_index: int, cm: bool = None):
        lib = nat.load()
        if cm is None:
            # measured: no gain on the headline's turn kernel (1.1654 vs 1.1656 ms; its FFMA2s
            # are mostly the forward half's), so off by default
            cm = CTAU and os.environ.get("QF_CTAU_TURN", "0") not in ("0", "", "false")
        src, self.nt, self.smem = generate_turn(fwd, adj, cm=cm)
        img = compile_kernel(src, "qf_turn")
        self.module = C.c_void_p()
        nat.check(lib.qf_jit_load(img, C.byref(self.module)))
        f = C.c_void_p()
        nat.check(lib.qf_jit_function(self.module, b"qf_turn", max(self.smem, 48 * 1024), C.byref(f)))
        self.func = (C.c_void_p * 1)(f.value)
        self.fwd, self.adj = fwd, adj
        self.rows_shift = fwd.n - fwd.L
        self.device_index = device_index
        self._slabs, self._plain = None, None
        if src.startswith("// QF_CM_COLS "):
            cols = [int(x) for x in src.split("\n", 1)[0].split()[2].split(",")]
            self._slabs = _SlabModules([img], ["qf_turn"], [(self.nt, self.smem)], [cols], b"qf_cm_a",
                                       device_index, [self.module], [f.value])

    def run(self, rows, psi_src, mats_f, angles_f, coefs_f, partials_f, lam, mats_a, angles_a, coefs_a,
            coef_stride_a, partials_a, stream):
        lib = nat.load()
        f, a = self.fwd, self.adj
        args = QfTurnArgs(
            a=QfJitArgs(psi=psi_src, lam=0, mats=mats_f, angles=angles_f, coefs=coefs_f, partials=partials_f,
                        n_mat=f.n_mat, n_ang=f.n_ang, coef_stride=0, n_slots=f.n_slots, tiles_log2=self.rows_shift,
                        pad=rows, psi_src=psi_src, skip_psi=0),
            b=QfJitArgs(psi=psi_src, lam=lam, mats=mats_a, angles=angles_a, coefs=coefs_a, partials=partials_a,
                        n_mat=a.n_mat, n_ang=a.n_ang, coef_stride=coef_stride_a, n_slots=a.n_slots,
                        tiles_log2=self.rows_shift, pad=rows, psi_src=0, skip_psi=1))
        grid = (C.c_uint32 * 1)(rows << self.rows_shift)
        block = (C.c_uint32 * 1)(self.nt)
        smem = (C.c_uint32 * 1)(self.smem)
        func = self.func
        if self._slabs is not None:
            if rows <= self._slabs.rows_max:
                func = self._slabs.stage(rows, mats_a, a.n_mat, stream, [0])
            else:   # more rows than the slab holds: the shared-memory variant (compiled once)
                if self._plain is None:
                    self._plain = TurnKernel(self.fwd, self.adj, self.device_index, cm=False)
                func = self._plain.func
        nat.check(lib.qf_jit_run(func, grid, block, smem, 1, stream, C.byref(args), C.sizeof(args)))


_OPTS = [b"--gpu-architecture=sm_100a", b"-std=c++17", b"-lineinfo", b"--device-as-default-execution-space"]
if os.environ.get("QF_GRAD_CHAINS"):
    _OPTS.append(f"-DGRAD_CHAINS={int(os.environ['QF_GRAD_CHAINS'])}".encode())


def _cache_dir() -> str:
    d = os.environ.get("QF_JIT_CACHE", os.path.join(os.path.expanduser("~"), ".cache", "qfb200"))
    os.makedirs(d, exist_ok=True)
    return d


def full_source(source: str) -> str:
    """Prelude + kernel body (QF_CM defined for modules with a constant-bank slab)."""
    return ("#define QF_CM 1\n" if "qf_cm_" in source else "") + prelude() + "\n" + source


def compile_kernel(source: str, name: str) -> bytes:
    """NVRTC-compile one kernel (prelude + body) to an sm_100a cubin, with a disk cache.
    QF_JIT_DUMP=dir writes the source as dir/<name>.cu (ncu --import-source resolves the
    -lineinfo file name relative to the working directory)."""
    full = full_source(source)
    dump = os.environ.get("QF_JIT_DUMP")
    if dump:
        os.makedirs(dump, exist_ok=True)
        with open(os.path.join(dump, name + ".cu"), "w") as f:
            f.write(full)
    key = hashlib.sha256(full.encode() + b"|".join(_OPTS)).hexdigest()
    path = os.path.join(_cache_dir(), key + ".cubin")
    if os.path.exists(path):
        with open(path, "rb") as f:
            return f.read()
    lib = nat.load()
    arr = (C.c_char_p * len(_OPTS))(*_OPTS)
    img = C.c_void_p()
    size = C.c_size_t()
    nat.check(lib.qf_jit_compile(full.encode(), (name + ".cu").encode(), arr, len(_OPTS), C.byref(img),
                                 C.byref(size)))
    image = C.string_at(img, size.value)
    lib.qf_jit_free(img)
    tmp = path + f".{os.getpid()}.tmp"
    with open(tmp, "wb") as f:
        f.write(image)
    os.replace(tmp, path)
    return image


# Owner of the slab copies a thread's launches use: None = the launch stream; a CUDA graph being
# captured sets its own token (slab_owner), so the graph's kernel nodes point into module copies
# no stream -- and no other graph -- ever writes, pinned until release_slab_owner(token).
_SLAB_OWNER = threading.local()
_SLAB_SETS = weakref.WeakSet()


class slab_owner:
    """Context: this thread's constant-slab launches use module copies owned by ``token``."""

    def __init__(self, token):
        self.token = token

    def __enter__(self):
        self.prev = getattr(_SLAB_OWNER, "token", None)
        _SLAB_OWNER.token = self.token

    def __exit__(self, *exc):
        _SLAB_OWNER.token = self.prev


def release_slab_owner(token) -> None:
    """Unload the module copies pinned for ``token`` (its graph is gone)."""
    for sm in list(_SLAB_SETS):
        sm.release(("owner", token))


class _SlabModules:
    """Per-stream loaded copies of kernel modules with constant slabs (CTAU).

    A module's __constant__ slab is shared by every launch of that module, so each stream (and
    each CUDA graph, through slab_owner) gets its own loaded copy of the modules: stream order
    then keeps a slab write behind the launches that read the previous contents.  Stream copies
    are bounded (oldest dropped after a device sync); graph-owned copies stay until released."""

    def __init__(self, images, names, geo, cols, sym, device_index, base_modules, base_funcs):
        self.images, self.names, self.geo, self.cols, self.sym = images, names, geo, cols, sym
        self.k = [len(c) if c else 0 for c in cols]
        self.rows_max = CM_CAP // max(self.k)
        self.device_index = device_index
        self.base = (list(base_modules), list(base_funcs))
        self.inst = {}
        self.lock = threading.Lock()
        self.cols_t = None
        _SLAB_SETS.add(self)

    def release(self, key):
        import torch

        with self.lock:
            old = self.inst.pop(key, None)
            if old is None:
                return
            torch.cuda.synchronize(torch.device("cuda", self.device_index))
            lib = nat.load()
            for m in old[2]:
                if all(m is not b for b in self.base[0]):
                    lib.qf_jit_unload(m)

    def instance(self, stream):
        token = getattr(_SLAB_OWNER, "token", None)
        key = ("owner", token) if token is not None else int(stream or 0)
        inst = self.inst.get(key)
        if inst is not None:
            return inst
        import torch

        lib = nat.load()
        with self.lock:
            inst = self.inst.get(key)
            if inst is not None:
                return inst
            dev = torch.device("cuda", self.device_index)
            if self.cols_t is None:
                self.cols_t = [torch.tensor(c, dtype=torch.int32, device=dev) if c else None for c in self.cols]
            streams = [k for k in self.inst if not isinstance(k, tuple)]
            if len(streams) >= CM_MAX_COPIES:
                # bounded: drop the oldest stream copy once the device has drained its launches
                old = self.inst.pop(streams[0])
                torch.cuda.synchronize(dev)
                for m in old[2]:
                    if all(m is not b for b in self.base[0]):
                        lib.qf_jit_unload(m)
            if not any(inst_[2] is self.base[0] for inst_ in self.inst.values()):
                mods, funcs = self.base
            else:
                mods, funcs = [], []
                for img, nm, (_, smem) in zip(self.images, self.names, self.geo):
                    mod = C.c_void_p()
                    nat.check(lib.qf_jit_load(img, C.byref(mod)))
                    f = C.c_void_p()
                    nat.check(lib.qf_jit_function(mod, nm.encode(), max(smem, 48 * 1024), C.byref(f)))
                    mods.append(mod)
                    funcs.append(f.value)
            slabs = []
            for mod, c in zip(mods, self.cols):
                if not c:
                    slabs.append(None)
                    continue
                ptr, size = C.c_void_p(), C.c_size_t()
                nat.check(lib.qf_jit_global(mod, self.sym, C.byref(ptr), C.byref(size)))
                slabs.append((ptr.value, size.value, torch.empty(2 * CM_CAP, dtype=torch.float32, device=dev)))
            inst = ((C.c_void_p * len(funcs))(*funcs), slabs, mods)
            self.inst[key] = inst
        return inst

    def stage(self, rows, mats, n_mat, stream, which):
        """Gather the launch's coefficients into the stream's slabs; returns its function array."""
        if rows > self.rows_max:
            raise ValueError(f"{rows} rows exceed the constant slabs ({self.rows_max} rows)")
        funcs, slabs, _ = self.instance(stream)
        lib = nat.load()
        for i in which:
            if slabs[i] is None:
                continue
            sym, size, staging = slabs[i]
            nat.check(lib.qf_jit_cm_stage(mats, n_mat, rows, self.cols_t[i].data_ptr(), self.k[i],
                                          staging.data_ptr(), sym, size, stream))
        return funcs


class JitProgram:
    """Compiled, loaded kernels of one planner.Program (one module per pass, compiled in parallel)."""

    def __init__(self, prog: pl.Program, device_index: int, cm: bool = False):
        from concurrent.futures import ThreadPoolExecutor

        lib = nat.load()
        tag = "a" if prog.adjoint else "f"
        sources, names, geo = generate(prog, tag, cm=cm)
        with ThreadPoolExecutor(max_workers=min(len(sources), os.cpu_count() or 4)) as ex:
            images = list(ex.map(lambda a: compile_kernel(*a), zip(sources, names)))
        self.modules, funcs = [], []
        for img, nm, (_, smem) in zip(images, names, geo):
            mod = C.c_void_p()
            nat.check(lib.qf_jit_load(img, C.byref(mod)))
            f = C.c_void_p()
            nat.check(lib.qf_jit_function(mod, nm.encode(), max(smem, 48 * 1024), C.byref(f)))
            self.modules.append(mod)
            funcs.append(f.value)
        P = len(names)
        # constant slabs (CTAU): per pass the slab columns; a module's __constant__ array is
        # shared by every launch of that module, so each stream gets its own loaded copy of
        # the modules (stream order then keeps a slab write behind the launches reading it)
        self.cm_sym = f"qf_cm_{tag}".encode()
        self.cm_cols, self.cm_k = [], []
        self.device_index = device_index
        for s_ in sources:
            cols = None
            if s_.startswith("// QF_CM_COLS "):
                cols = [int(x) for x in s_.split("\n", 1)[0].split()[2].split(",")]
            self.cm_cols.append(cols)
            self.cm_k.append(len(cols) if cols else 0)
        self.cm = any(self.cm_k)
        self.cm_rows_max = CM_CAP // max(self.cm_k) if self.cm else 1 << 62
        self._images, self._names, self._geo = images, names, geo
        self.n = P
        self.names = names
        self.funcs = (C.c_void_p * P)(*funcs)
        self._slabs = _SlabModules(images, names, geo, self.cm_cols, self.cm_sym, device_index,
                                   self.modules[:P], funcs) if self.cm else None
        self.rows_shift = prog.n - prog.L
        self.block = (C.c_uint32 * P)(*[g[0] for g in geo])
        self.smem = (C.c_uint32 * P)(*[g[1] for g in geo])
        self.prog = prog
        self._remote = {}
        self.persist = PERSIST
        sms = lib.qf_device_sm_count(device_index)
        self.resident = []
        for f, (nt, smem) in zip(funcs, geo):
            occ = C.c_int(0)
            nat.check(lib.qf_jit_occupancy(f, nt, smem, C.byref(occ)))
            self.resident.append(max(1, occ.value) * max(1, sms))

    def _funcs_for(self, rows, mats, stream, which):
        """Function array for this launch; with constant slabs, stage passes ``which`` first."""
        if not self.cm:
            return self.funcs
        return self._slabs.stage(rows, mats, self.prog.n_mat, stream, which)

    def remote_pass(self, g: int):
        """(function, block, smem) of the last pass with the fused swap store (compiled once per g)."""
        hit = self._remote.get(g)
        if hit is None:
            lib = nat.load()
            tag = "a" if self.prog.adjoint else "f"
            srcs, names, geo = generate(self.prog, tag, remote_pass=len(self.prog.passes) - 1, remote_g=g)
            img = compile_kernel(srcs[0], names[0] + f"_g{g}")
            mod = C.c_void_p()
            nat.check(lib.qf_jit_load(img, C.byref(mod)))
            f = C.c_void_p()
            nat.check(lib.qf_jit_function(mod, names[0].encode(), max(geo[0][1], 48 * 1024), C.byref(f)))
            self.modules.append(mod)
            hit = self._remote[g] = (f.value, geo[0][0], geo[0][1])
        return hit

    def run_ckpt(self, rows, psis, srcs, lam, mats, angles, coefs, coef_stride, partials, stream, skip_psi,
                 which=None, tcb=0, tc_n=0):
        """One launch per pass with its own state pointers: psis[i] is pass i's state buffer,
        srcs[i] (forward) the buffer it loads from (0 = psis[i]); skip_psi: adjoint passes
        read psi from forward checkpoints and do not write it back."""
        lib = nat.load()
        which = range(self.n) if which is None else which
        funcs = self._funcs_for(rows, mats, stream, which)
        for i in which:
            args = QfJitArgs(psi=psis[i], lam=lam, mats=mats, angles=angles, coefs=coefs, partials=partials,
                             n_mat=self.prog.n_mat, n_ang=self.prog.n_ang, coef_stride=coef_stride,
                             n_slots=self.prog.n_slots, tiles_log2=self.rows_shift, pad=rows,
                             psi_src=srcs[i] if srcs else 0, skip_psi=int(bool(skip_psi)), tcb=tcb, tc_n=tc_n)
            total = rows << self.rows_shift
            # a per-call grid array: JitPrograms are shared across threads and batch sizes
            grid = (C.c_uint32 * 1)(min(total, self.resident[i]) if self.persist else total)
            nat.check(lib.qf_jit_run(C.addressof(funcs) + C.sizeof(C.c_void_p) * i,
                                     grid, C.addressof(self.block) + 4 * i,
                                     C.addressof(self.smem) + 4 * i, 1, stream, C.byref(args), C.sizeof(args)))

    def run(self, rows, psi, lam, mats, angles, coefs, coef_stride, partials, stream, first=0, last=None,
            remote=None, tcb=0, tc_n=0):
        """remote = (device array of the ranks' receive-shard pointers, rank of row 0, g): the
        last pass writes its output into those shards (a fused global-qubit swap)."""
        lib = nat.load()
        last = self.n if last is None else last
        args = QfJitArgs(psi=psi, lam=lam, mats=mats, angles=angles, coefs=coefs, partials=partials,
                         n_mat=self.prog.n_mat, n_ang=self.prog.n_ang, coef_stride=coef_stride,
                         n_slots=self.prog.n_slots, tiles_log2=self.rows_shift, pad=rows, tcb=tcb, tc_n=tc_n)
        if remote is not None:
            peers, rank_base, g = remote
            args.peers, args.rank_base = peers, rank_base
            if last == self.n:
                if last - 1 > first:
                    self.run(rows, psi, lam, mats, angles, coefs, coef_stride, partials, stream, first, last - 1,
                             tcb=tcb, tc_n=tc_n)
                f, nt, smem = self.remote_pass(g)
                funcs = (C.c_void_p * 1)(f)
                grid = (C.c_uint32 * 1)(rows << self.rows_shift)
                block = (C.c_uint32 * 1)(nt)
                sm = (C.c_uint32 * 1)(smem)
                nat.check(lib.qf_jit_run(funcs, grid, block, sm, 1, stream, C.byref(args), C.sizeof(args)))
                return
        total = rows << self.rows_shift
        cnt = last - first
        # a per-call grid array: JitPrograms are shared across threads and batch sizes
        grid = (C.c_uint32 * cnt)(*[min(total, self.resident[i]) if self.persist else total
                                    for i in range(first, last)])
        funcs = self._funcs_for(rows, mats, stream, range(first, last))
        nat.check(lib.qf_jit_run(C.addressof(funcs) + C.sizeof(C.c_void_p) * first,
                                 grid, C.addressof(self.block) + 4 * first,
                                 C.addressof(self.smem) + 4 * first, cnt, stream, C.byref(args), C.sizeof(args)))


def enabled(rows: int, n_eff: int) -> bool:
    """Plan-specialised kernels pay off once a launch moves enough data to amortise the
    one-off NVRTC compile; QF_JIT=1/0 forces them on/off."""
    flag = os.environ.get("QF_JIT")
    if flag is not None:
        return flag not in ("0", "", "false", "no")
    return rows * (1 << n_eff) >= (1 << 20)   # cfg1 (1024 x 2^10): 1.85x faster than interpreted
