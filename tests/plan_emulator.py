"""NumPy emulator of a planner.Program (test infrastructure).

Executes the exact descriptor arrays the CUDA kernels consume -- build recipe,
passes, stages, ops, term tables, subset tables, gradient slots -- but on the
whole state vector at once, so the planner / emitter can be verified on the CPU
against the oracle.  It also checks the invariants the kernels rely on (terms
grouped by register subset, dense ops on register slots with s0 < s1, lanes on
qubits 0..4 at load/store).
"""

from __future__ import annotations

import numpy as np

from paper_2003_02989_b200 import planner as pl


def build_tables(prog: pl.Program, theta: np.ndarray, fixed: np.ndarray, consts: np.ndarray):
    r = prog.recipe
    B = theta.shape[0]
    gen_ev = r["gen_eval"].reshape(-1, 4)
    gen_vec = r["gen_evec"].reshape(-1, 4, 4, 2)
    gen_vec = gen_vec[..., 0] + 1j * gen_vec[..., 1]
    mats = np.zeros((B, max(prog.n_mat, 1)), dtype=np.complex128)
    angs = np.zeros((B, max(prog.n_ang, 1)), dtype=np.float64)
    sg = [0, 2, 1, 3]

    def gen_mat(b, g):
        d = r["gen_dim"][g]
        v = r["gen_coeff"][g] * float(theta[b, r["gen_sym"][g]]) + r["gen_const"][g]
        V = gen_vec[g, :d, :d]
        m = np.zeros((4, 4), dtype=np.complex128)
        m[:d, :d] = (V * np.exp(-1j * v * gen_ev[g, :d])) @ V.conj().T
        return m

    for b in range(B):
        for i, off in enumerate(r["dense_mat"]):
            D = r["dense_dim"][i]
            M = np.eye(D, dtype=np.complex128)
            for f in range(r["dense_fbeg"][i], r["dense_fbeg"][i + 1]):
                kind, src, emb = r["factor"][3 * f: 3 * f + 3]
                F = gen_mat(b, src) if kind == 0 else fixed[b if fixed.shape[0] > 1 else 0, src]
                if emb == 4:
                    G = F[:2, :2]
                elif emb == 0:
                    G = F
                elif emb == 1:
                    G = F[np.ix_(sg, sg)]
                elif emb == 2:
                    G = np.kron(F[:2, :2], np.eye(2))
                else:
                    G = np.kron(np.eye(2), F[:2, :2])
                M = G @ M
            mats[b, off:off + D * D] = M.reshape(-1)
        for k in range(len(r["term_beta"])):
            kind, src = r["term_src"][2 * k: 2 * k + 2]
            if kind == 0:
                v = r["gen_coeff"][src] * float(theta[b, r["gen_sym"][src]]) + r["gen_const"][src]
                angs[b, k] = v * r["term_beta"][k]
            else:
                angs[b, k] = consts[b if consts.shape[0] > 1 else 0, src]
    return mats, angs


def _apply(psi, m, qs, n):
    k = len(qs)
    full = psi.reshape((2,) * n)
    axes = [n - 1 - q for q in qs]
    out = np.tensordot(m.reshape((2,) * (2 * k)), full, axes=(list(range(k, 2 * k)), axes))
    out = np.moveaxis(out, list(range(k)), axes)
    return np.ascontiguousarray(out).reshape(-1)


def _chi(idx, mask):
    par = np.zeros_like(idx)
    m = int(mask)
    while m:
        low = m & -m
        par ^= (idx & low) != 0
        m ^= low
    return 1.0 - 2.0 * par


def _q1(o, st, reg_glob):
    """Physical qubit of a one-qubit op: its register slot, or (lane op) its thread bit."""
    return int(st[8 + o[15] - 1]) if o[15] else reg_glob[o[1]]


def check_invariants(prog: pl.Program):
    R = prog.R
    for p in prog.passes:
        sb, se = p[0], p[1]
        for si in range(sb, se):
            st = prog.stages[si]
            reg_glob = list(st[0:R])
            lanes = list(st[8:12])
            vec = int(st[0]) == 0       # 16-byte edge layout: qubit 0 in register slot 0
            edge = [1, 2, 3, 4] if vec else [0, 1, 2, 3]
            if si == sb:
                assert lanes == edge, (si, lanes)
            if si == se - 1:
                if p[126]:   # relabelled: the store lanes are the bits stored to physical 0..3
                    outer = set(int(x) for x in p[16:16 + p[10]])
                    tileq = [q for q in range(prog.n) if q not in outer]
                    out_of = {tileq[i]: int(p[84 + i]) for i in range(len(tileq))}
                    assert [out_of[int(x)] for x in lanes] == [0, 1, 2, 3], (si, lanes)
                else:
                    assert lanes == edge, (si, lanes)
            for o in prog.ops[st[48]:st[49]]:
                if o[0] == pl.OP_DENSE2:
                    assert 0 <= o[1] < o[2] < R
                if o[0] == pl.OP_DENSE1:
                    assert (o[1] == -1 and 1 <= o[15] <= 5) if o[15] else 0 <= o[1] < R
                if o[0] in (pl.OP_DIAG, pl.OP_OBS):
                    g = prog.grp[o[6]: o[6] + (1 << R) + 1]
                    for S in range(1 << R):
                        for k in range(g[S], g[S + 1]):
                            assert pl._bit_subset(int(prog.term_mask[k]), reg_glob) == S


def run_forward(prog: pl.Program, mats, angs, B, n, coefs=None, init_state=None):
    dim = 1 << n
    idx = np.arange(dim)
    psi = np.zeros((B, dim), dtype=np.complex128)
    slots = np.zeros((B, max(prog.n_slots, 1)))
    for b in range(B):
        for pi, p in enumerate(prog.passes):
            if p[2] == pl.INIT_ZERO:
                psi[b] = 0
                psi[b, 0] = 1
            elif p[2] == pl.INIT_PRODUCT:
                st = np.ones(1, dtype=np.complex128)
                for q in range(n - 1, -1, -1):
                    mo = p[48 + q]
                    f = np.array([1, 0], dtype=np.complex128) if mo < 0 else mats[b, [mo, mo + 2]]
                    st = np.kron(st, f)
                psi[b] = st
            for si in range(p[0], p[1]):
                st = prog.stages[si]
                reg_glob = list(st[0:prog.R])
                for o in prog.ops[st[48]:st[49]]:
                    if o[0] == pl.OP_DENSE1:
                        psi[b] = _apply(psi[b], mats[b, o[3]:o[3] + 4].reshape(2, 2), [_q1(o, st, reg_glob)], n)
                    elif o[0] == pl.OP_DENSE2:
                        psi[b] = _apply(psi[b], mats[b, o[3]:o[3] + 16].reshape(4, 4),
                                        [reg_glob[o[1]], reg_glob[o[2]]], n)
                    elif o[0] == pl.OP_DIAG:
                        ang = np.zeros(dim)
                        for k in range(o[4], o[5]):
                            ang += angs[b, prog.term_idx[k]] * _chi(idx, prog.term_mask[k])
                        psi[b] = psi[b] * np.exp(-1j * ang)
                    elif o[0] == pl.OP_OBS:
                        h = np.zeros(dim)
                        for k in range(o[4], o[5]):
                            h += coefs[-1 - prog.term_idx[k]] * _chi(idx, prog.term_mask[k])
                        slots[b, o[7]] += float(np.sum(np.abs(psi[b]) ** 2 * h))
            if p[126]:      # relabelled store: tile bit at physical tileq[i] goes to p[84 + i]
                outer = set(int(x) for x in p[16:16 + p[10]])
                tileq = [q for q in range(n) if q not in outer]
                psi[b] = permute_bits(psi[b], {tileq[i]: int(p[84 + i]) for i in range(len(tileq))}, n)
    return psi, slots


def permute_bits(v, perm: dict, n: int):
    """out[j] = v[i] where bit perm[a] of j is bit a of i (bits not in perm stay)."""
    idx = np.arange(1 << n)
    j = idx.copy()
    for a, b in perm.items():
        j &= ~(1 << b)
    for a, b in perm.items():
        j |= ((idx >> a) & 1) << b
    out = np.empty_like(v)
    out[j] = v
    return out


def logical_state(psi, prog: pl.Program, n: int):
    """A relabelled program's output in the logical layout (physical bit final_pos[q] = qubit q)."""
    if prog.final_pos is None:
        return psi
    inv = {prog.final_pos[q]: q for q in range(n)}
    return np.stack([permute_bits(row, inv, n) for row in psi])


def run_adjoint(prog: pl.Program, mats, angs, B, n, psi, lam, hcoefs):
    """Backward program on (psi, lam) (lam ignored when the first pass seeds it)."""
    dim = 1 << n
    idx = np.arange(dim)
    psi = psi.copy()
    lam = lam.copy() if lam is not None else np.zeros_like(psi)
    slots = np.zeros((B, max(prog.n_slots, 1)))
    gm = prog.genmats.reshape(-1, 2)
    gm = gm[:, 0] + 1j * gm[:, 1]
    for b in range(B):
        for p in prog.passes:
            for si in range(p[0], p[1]):
                st = prog.stages[si]
                reg_glob = list(st[0:prog.R])
                for o in prog.ops[st[48]:st[49]]:
                    if o[0] in (pl.OP_DENSE1, pl.OP_DENSE2):
                        qs = [_q1(o, st, reg_glob)] if o[0] == pl.OP_DENSE1 else [reg_glob[o[1]], reg_glob[o[2]]]
                        d = 1 << len(qs)
                        u = mats[b, o[3]:o[3] + d * d].reshape(d, d)
                        if o[13]:   # fused block: U^dag, then the two-point matrix A (slots)
                            psi[b] = _apply(psi[b], u.conj().T, qs, n)
                            lam[b] = _apply(lam[b], u.conj().T, qs, n)
                            slots[b, o[7]:o[7] + d * d] += _block_a(psi[b], lam[b], qs, n)
                            continue
                        if o[7] >= 0:
                            g = gm[o[8]:o[8] + d * d].reshape(d, d)
                            slots[b, o[7]] += float(np.vdot(lam[b], _apply(psi[b], g, qs, n)).imag)
                        psi[b] = _apply(psi[b], u.conj().T, qs, n)
                        lam[b] = _apply(lam[b], u.conj().T, qs, n)
                    elif o[0] == pl.OP_DIAG:
                        ang = np.zeros(dim)
                        wsum = np.zeros(dim)
                        for k in range(o[4], o[5]):
                            chi = _chi(idx, prog.term_mask[k])
                            ang += angs[b, prog.term_idx[k]] * chi
                            wsum += prog.term_w[k] * chi
                        if o[7] >= 0:
                            slots[b, o[7]] += float(np.sum(wsum * (lam[b].conj() * psi[b]).imag))
                        ph = np.exp(1j * ang)
                        psi[b] *= ph
                        lam[b] *= ph
                    elif o[0] == pl.OP_OBS:
                        h = np.zeros(dim)
                        for k in range(o[4], o[5]):
                            h += hcoefs[b, -1 - prog.term_idx[k]] * _chi(idx, prog.term_mask[k])
                        lam[b] = h * psi[b]
                        slots[b, o[7]] += float(np.sum(np.abs(psi[b]) ** 2 * h))
    return slots


def _block_a(psi, lam, qs, n):
    """A = (rho - rho^dag)/2i, rho[j][k] = sum psi_j conj(lam_k), in qf_block_grads' slot
    order (diagonal, then 2 Re / 2 Im of the upper entries)."""
    d = 1 << len(qs)
    p = np.moveaxis(psi.reshape((2,) * n), [n - 1 - q for q in qs], list(range(len(qs)))).reshape(d, -1)
    l = np.moveaxis(lam.reshape((2,) * n), [n - 1 - q for q in qs], list(range(len(qs)))).reshape(d, -1)
    rho = p @ l.conj().T
    A = (rho - rho.conj().T) / 2j
    out = [A[j, j].real for j in range(d)]
    for j in range(d):
        for k in range(j + 1, d):
            out += [2 * A[j, k].real, 2 * A[j, k].imag]
    return np.array(out)


def block_grads(prog: pl.Program, mats, a_slots, n_cols):
    """NumPy restatement of qf_block_grads: per factor Tr(W^dag G W A), summed per symbol."""
    B = a_slots.shape[0]
    out = np.zeros((B, n_cols))
    gens = prog.block_gens.reshape(-1, 2)
    gens = gens[:, 0] + 1j * gens[:, 1]
    for b in range(B):
        for fb, fe, D, slot0 in prog.blocks:
            a = a_slots[b, slot0:slot0 + D * D]
            A = np.zeros((D, D), dtype=np.complex128)
            e = D
            for j in range(D):
                A[j, j] = a[j]
                for k in range(j + 1, D):
                    A[j, k] = (a[e] + 1j * a[e + 1]) / 2
                    A[k, j] = np.conj(A[j, k])
                    e += 2
            W = np.eye(D, dtype=np.complex128)
            for moff, goff, sym in prog.block_factors[fb:fe]:
                W = mats[b, moff:moff + D * D].reshape(D, D) @ W
                if goff >= 0:
                    G = gens[goff:goff + D * D].reshape(D, D)
                    out[b, sym] += float(np.trace(W.conj().T @ G @ W @ A).real)
    return out


def slots_to_cols(slots, mapping, n_cols):
    out = np.zeros((slots.shape[0], n_cols))
    for c, ss in mapping.items():
        for s in ss:
            out[:, c] += slots[:, s]
    return out
