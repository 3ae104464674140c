// Tile-pass kernels: one CTA = one (row, tile) of 2^L amplitudes; each thread keeps
// 2^R amplitudes in registers.  A pass applies a whole run of fused gates whose
// targets lie inside the tile's qubit set Q (|Q| = L, Q contains qubits 0..4 so
// every warp-wide global access is 256 contiguous bytes).  Within a pass the
// planner splits the op list into stages; each stage has a register mapping
// (which tile bits live in registers) and consecutive stages are connected by one
// swizzled shared-memory transpose.  Diagonal gates are phase polynomials
// evaluated from the amplitude index (integer Walsh-Hadamard transform over the
// register bits) and need no data movement.
//
// Reference semantics accelerated here: qcflow/sim.py:88-136 (apply_matrix /
// run_ops), sim.py:177-213 (Pauli expectation); the ADJ instantiation is the
// adjoint differentiator whose oracle is gradients.py:158-165 / :241-326.
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "qf_common.cuh"

namespace qf {

template <int N, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  [&]<int... I>(std::integer_sequence<int, I...>) {
    (f(std::integral_constant<int, I>{}), ...);
  }(std::make_integer_sequence<int, N>{});
}

// Visit the 2^R register indices in Gray-code order with a running XOR offset
// (consecutive Gray codes differ in one bit -> one LOP per amplitude).
template <int R, typename F>
__device__ __forceinline__ void gray_walk(uint32_t base, const uint32_t (&step)[R], F&& f) {
  uint32_t off = base;
  static_for<(1 << R)>([&](auto I) {
    constexpr int i = decltype(I)::value;
    if constexpr (i != 0) {
      constexpr int j = ctz_c(i);
      off ^= step[j];
    }
    f(std::integral_constant<int, gray_c(i)>{}, off);
  });
}

// ---------------------------------------------------------------------------
// dense gates on register slots (compile-time slots, runtime matrices in smem)
// ---------------------------------------------------------------------------

// U (2x2) on register slot J; CLS selects the arithmetic for the matrix structure
// (0 general complex, 1 [[a, ib], [ic, d]], 2 real) -- 4 / 2 / 2 FP32x2 ops per amplitude.
template <int J, int NR, int CLS>
__device__ __forceinline__ void apply1(float2 (&v)[NR], float2 u00, float2 u01, float2 u10, float2 u11) {
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    if (r & (1 << J)) continue;
    const float2 a = v[r], b = v[r | (1 << J)];
    if constexpr (CLS == 0) {
      v[r] = cmad2(u00, a, u01, b);
      v[r | (1 << J)] = cmad2(u10, a, u11, b);
    } else if constexpr (CLS == 1) {
      v[r] = xrow(u00.x, a, u01.y, b);
      v[r | (1 << J)] = xrow(u11.x, b, u10.y, a);
    } else {
      v[r] = rrow(u00.x, a, u01.x, b);
      v[r | (1 << J)] = rrow(u10.x, a, u11.x, b);
    }
  }
}

// load a 2x2 from smem, optionally as its conjugate transpose
__device__ __forceinline__ void load_u2(const float2* u, bool adj, float2& u00, float2& u01, float2& u10,
                                        float2& u11) {
  u00 = u[0];
  u01 = u[1];
  u10 = u[2];
  u11 = u[3];
  if (adj) {
    const float2 t = u01;
    u00.y = -u00.y;
    u11.y = -u11.y;
    u01 = make_float2(u10.x, -u10.y);
    u10 = make_float2(t.x, -t.y);
  }
}

template <int J0, int J1, int NR>
__device__ __forceinline__ void apply2(float2 (&v)[NR], const float2* __restrict__ u, bool adj) {
  float2 m[16];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 x = adj ? u[j * 4 + i] : u[i * 4 + j];
      if (adj) x.y = -x.y;
      m[i * 4 + j] = x;
    }
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    if (r & ((1 << J0) | (1 << J1))) continue;
    const int i0 = r, i1 = r | (1 << J1), i2 = r | (1 << J0), i3 = r | (1 << J0) | (1 << J1);
    const float2 a0 = v[i0], a1 = v[i1], a2 = v[i2], a3 = v[i3];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 o = cmad2(m[i * 4 + 0], a0, m[i * 4 + 1], a1);
      o = cfma(m[i * 4 + 2], a2, o);
      o = cfma(m[i * 4 + 3], a3, o);
      v[i == 0 ? i0 : i == 1 ? i1 : i == 2 ? i2 : i3] = o;
    }
  }
}

// Im <lam| G |psi> over the register pairs of slot J (G Hermitian 2x2).
template <int J, int NR>
__device__ __forceinline__ float grad1(const float2 (&p)[NR], const float2 (&l)[NR], const float2* g) {
  const float2 g00 = g[0], g01 = g[1], g10 = g[2], g11 = g[3];
  float acc = 0.f;
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    if (r & (1 << J)) continue;
    const int r1 = r | (1 << J);
    const float2 t0 = cmad2(g00, p[r], g01, p[r1]);
    const float2 t1 = cmad2(g10, p[r], g11, p[r1]);
    acc += im_conj_mul(l[r], t0) + im_conj_mul(l[r1], t1);
  }
  return acc;
}

// Im <lam| c P |psi> for a single Pauli P on slot J (GK 1 = X, 2 = Y, 3 = Z); c applied by the caller.
template <int J, int NR, int GK>
__device__ __forceinline__ float gradp(const float2 (&p)[NR], const float2 (&l)[NR]) {
  float acc = 0.f;
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    if (r & (1 << J)) continue;
    const int r1 = r | (1 << J);
    if constexpr (GK == 1) {
      acc += im_conj_mul(l[r], p[r1]) + im_conj_mul(l[r1], p[r]);
    } else if constexpr (GK == 2) {
      acc += re_conj_mul(l[r1], p[r]) - re_conj_mul(l[r], p[r1]);
    } else {
      acc += im_conj_mul(l[r], p[r]) - im_conj_mul(l[r1], p[r1]);
    }
  }
  return acc;
}

template <int J0, int J1, int NR>
__device__ __forceinline__ float grad2(const float2 (&p)[NR], const float2 (&l)[NR], const float2* g) {
  float acc = 0.f;
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    if (r & ((1 << J0) | (1 << J1))) continue;
    const int idx[4] = {r, r | (1 << J1), r | (1 << J0), r | (1 << J0) | (1 << J1)};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 t = cmad2(g[i * 4 + 0], p[idx[0]], g[i * 4 + 1], p[idx[1]]);
      const float2 u = cmad2(g[i * 4 + 2], p[idx[2]], g[i * 4 + 3], p[idx[3]]);
      t.x += u.x;
      t.y += u.y;
      acc += im_conj_mul(l[idx[i]], t);
    }
  }
  return acc;
}

// dispatch a runtime register slot onto compile-time instantiations
template <int R, typename Fn>
__device__ __forceinline__ void dispatch1(int s, Fn&& fn) {
  switch (s) {
    case 0: if constexpr (0 < R) fn.template operator()<0>(); break;
    case 1: if constexpr (1 < R) fn.template operator()<1>(); break;
    case 2: if constexpr (2 < R) fn.template operator()<2>(); break;
    case 3: if constexpr (3 < R) fn.template operator()<3>(); break;
    case 4: if constexpr (4 < R) fn.template operator()<4>(); break;
    case 5: if constexpr (5 < R) fn.template operator()<5>(); break;
    default: break;
  }
}

template <int R, typename Fn>
__device__ __forceinline__ void dispatch2(int s0, int s1, Fn&& fn) {
#define QF_P(A, B)                                                \
  case A * 8 + B:                                                 \
    if constexpr (A < R && B < R) fn.template operator()<A, B>(); \
    break;
  switch (s0 * 8 + s1) {
    QF_P(0, 1) QF_P(0, 2) QF_P(0, 3) QF_P(0, 4) QF_P(0, 5)
    QF_P(1, 2) QF_P(1, 3) QF_P(1, 4) QF_P(1, 5)
    QF_P(2, 3) QF_P(2, 4) QF_P(2, 5)
    QF_P(3, 4) QF_P(3, 5)
    QF_P(4, 5)
    default: break;
  }
#undef QF_P
}

// ---------------------------------------------------------------------------
// stage geometry
// ---------------------------------------------------------------------------

// XOR of per-thread-bit contributions (global bit positions or swizzled smem offsets).
template <int TB>
__device__ __forceinline__ uint32_t thread_glob(const QfStage& st, int t) {
  uint32_t x = 0;
#pragma unroll
  for (int i = 0; i < TB; ++i)
    if (t & (1 << i)) x ^= 1u << st.thr_glob[i];
  return x;
}
template <int TB>
__device__ __forceinline__ uint32_t thread_phys(const QfStage& st, int t) {
  uint32_t x = 0;
#pragma unroll
  for (int i = 0; i < TB; ++i)
    if (t & (1 << i)) x ^= (uint32_t)st.thr_phys[i];
  return x;
}

// write v (mapping `from`) to smem, read back with mapping `to`.
template <int R, int TB, int NA>
__device__ __forceinline__ void remap(float2 (&v)[NA][1 << R], float2* sm, const QfStage& from,
                                      const QfStage& to, int t) {
  constexpr int TILE = 1 << (R + TB);
  uint32_t ph[R];
  __syncthreads();
#pragma unroll
  for (int j = 0; j < R; ++j) ph[j] = (uint32_t)from.reg_phys[j];
  gray_walk<R>(thread_phys<TB>(from, t), ph, [&](auto r, uint32_t addr) {
#pragma unroll
    for (int q = 0; q < NA; ++q) sm[q * TILE + addr] = v[q][decltype(r)::value];
  });
  __syncthreads();
#pragma unroll
  for (int j = 0; j < R; ++j) ph[j] = (uint32_t)to.reg_phys[j];
  gray_walk<R>(thread_phys<TB>(to, t), ph, [&](auto r, uint32_t addr) {
#pragma unroll
    for (int q = 0; q < NA; ++q) v[q][decltype(r)::value] = sm[q * TILE + addr];
  });
}

// A[S] = sum_{k: subset(k) = S} (-1)^{popc(gt & mask_k)} * value_k
// grp: smem subset-boundary table (2^R + 1 entries, pass-relative term indices).
template <int R, typename T, typename ValFn>
__device__ __forceinline__ void subset_accumulate(T (&A)[1 << R], const int32_t* grp, const uint2* terms,
                                                  uint32_t gt, ValFn&& val) {
  static_for<(1 << R)>([&](auto SI) {
    constexpr int S = decltype(SI)::value;
    T acc = T(0);
    const int kb = grp[S], ke = grp[S + 1];
    for (int k = kb; k < ke; ++k) {
      const uint2 tm = terms[k];
      const T x = val(tm, k);
      acc = (__popc(gt & tm.x) & 1) ? acc - x : acc + x;
    }
    A[S] = acc;
  });
}

// ---------------------------------------------------------------------------
// the pass kernel
// ---------------------------------------------------------------------------

template <int L, int R, bool ADJ>
struct KTraits {
  static constexpr int NT = 1 << (L - R);
  // forward tiles of 8192 amplitudes fit two CTAs per SM at <=128 registers
  // at most 128 registers per thread: 65536 / (threads * 128) resident CTAs per SM
  static constexpr int MINB = (65536 / (NT * 128)) > 8 ? 8 : (65536 / (NT * 128));
};

template <int L, int R, bool ADJ>
__global__ void __launch_bounds__(KTraits<L, R, ADJ>::NT, KTraits<L, R, ADJ>::MINB) pass_kernel(const PassArgs a) {
  constexpr int NR = 1 << R;
  constexpr int TB = L - R;
  constexpr int NT = 1 << TB;
  constexpr int NA = ADJ ? 2 : 1;  // amplitude arrays (psi, lambda)
  constexpr int TILE = 1 << L;
  extern __shared__ __align__(16) unsigned char smem_raw[];

  const QfProgram& P = a.prog;
  const QfPass* gpass = P.passes + a.pass;
  const int t = threadIdx.x;
  const int tiles_log2 = a.tiles_log2;
  const int row = (int)(blockIdx.x >> tiles_log2);
  const uint32_t o = blockIdx.x & ((1u << tiles_log2) - 1u);

  const int mat_begin = gpass->mat_begin, mat_cnt = gpass->mat_end - mat_begin;
  const int term_begin = gpass->term_begin, term_cnt = gpass->term_end - term_begin;
  const int grp_begin = gpass->grp_begin, grp_cnt = gpass->grp_end - grp_begin;
  const int op_begin = gpass->op_begin, op_cnt = gpass->op_end - op_begin;
  const int st_begin = gpass->stage_begin, st_cnt = gpass->stage_end - st_begin;
  const int slot_begin = gpass->slot_begin, slot_cnt = gpass->slot_end - slot_begin;

  // ---- shared memory carve-up ----
  float2* tile = reinterpret_cast<float2*>(smem_raw);
  QfStage* sst = reinterpret_cast<QfStage*>(tile + NA * TILE);
  QfOp* sop = reinterpret_cast<QfOp*>(sst + st_cnt);
  // slot partials: one entry per (slot, warp), summed in warp order at the end, so results
  // are bit-identical from call to call (no shared-memory atomics)
  constexpr int NW = NT / 32;
  double* ssm = reinterpret_cast<double*>(sop + op_cnt);
  float2* msm = reinterpret_cast<float2*>(ssm + slot_cnt * NW);
  uint2* stm = reinterpret_cast<uint2*>(msm + mat_cnt);
  float* stw = reinterpret_cast<float*>(stm + term_cnt);
  int32_t* sgr = reinterpret_cast<int32_t*>(stw + (ADJ ? term_cnt : 0));

  {
    const int32_t* s32 = reinterpret_cast<const int32_t*>(P.stages + st_begin);
    int32_t* d32 = reinterpret_cast<int32_t*>(sst);
    for (int i = t; i < st_cnt * 64; i += NT) d32[i] = s32[i];
    s32 = reinterpret_cast<const int32_t*>(P.ops + op_begin);
    d32 = reinterpret_cast<int32_t*>(sop);
    for (int i = t; i < op_cnt * 16; i += NT) d32[i] = s32[i];
    for (int i = t; i < slot_cnt * NW; i += NT) ssm[i] = 0.0;
    const float2* src = a.mats + (size_t)row * P.n_mat + mat_begin;
    for (int i = t; i < mat_cnt; i += NT) msm[i] = src[i];
    const int32_t* arow = a.angles + (size_t)row * P.n_ang;
    const float* crow = a.coefs + (size_t)row * P.coef_row_stride;
    for (int i = t; i < term_cnt; i += NT) {
      const int k = term_begin + i;
      const int idx = P.term_idx[k];
      // DIAG terms index the angle table, OBS terms the coefficient table; the planner
      // marks OBS columns with a negative index (-1 - column).
      const int32_t val = idx >= 0 ? arow[idx] : __float_as_int(crow[-1 - idx]);
      stm[i] = make_uint2(P.term_mask[k], (uint32_t)val);
      if constexpr (ADJ) stw[i] = P.term_w[k];
    }
    for (int i = t; i < grp_cnt; i += NT) sgr[i] = P.grp[grp_begin + i] - term_begin;
  }

  // global bits of this tile's outer index
  uint32_t base = 0;
  {
    const int nout = gpass->n_outer;
    for (int i = 0; i < nout; ++i)
      if (o & (1u << i)) base |= 1u << gpass->outer_pos[i];
  }
  const int init = gpass->init, store = gpass->store;

  const size_t row_elems = (size_t)1 << a.n;
  float2* psi_row = a.psi + (size_t)row * row_elems;
  float2* lam_row = ADJ ? a.lam + (size_t)row * row_elems : nullptr;

  float2 v[NA][NR];
  __syncthreads();

  // ---- load / initialise (stage 0 mapping; lanes sit on qubits 0..4) ----
  {
    const QfStage& st0 = sst[0];
    const uint32_t gt = base | thread_glob<TB>(st0, t);
    uint32_t rg[R];
#pragma unroll
    for (int j = 0; j < R; ++j) rg[j] = 1u << st0.reg_glob[j];
    if (init == QF_INIT_LOAD || init == QF_INIT_LOAD_PSI) {
      const bool with_lam = ADJ && init == QF_INIT_LOAD;
      gray_walk<R>(gt, rg, [&](auto r, uint32_t g) {
        constexpr int ri = decltype(r)::value;
        v[0][ri] = psi_row[g];
        if constexpr (ADJ) v[1][ri] = with_lam ? lam_row[g] : make_float2(0.f, 0.f);
      });
    } else if (init == QF_INIT_ZERO) {
      gray_walk<R>(gt, rg, [&](auto r, uint32_t g) {
        constexpr int ri = decltype(r)::value;
        v[0][ri] = make_float2(g == 0 ? 1.f : 0.f, 0.f);
        if constexpr (ADJ) v[1][ri] = make_float2(0.f, 0.f);
      });
    } else {  // product state: amp(x) = prod_q f_q[bit_q(x)], f_q = column 0 of qubit q's leading 2x2
      float2 c = make_float2(1.f, 0.f);
      uint32_t regmask = 0;
#pragma unroll
      for (int j = 0; j < R; ++j) regmask |= rg[j];
      for (int q = 0; q < a.n; ++q) {
        if (regmask & (1u << q)) continue;
        const int mo = gpass->init_mat[q];
        const int bit = (gt >> q) & 1;
        const float2 f = mo < 0 ? make_float2(bit ? 0.f : 1.f, 0.f) : msm[mo - mat_begin + (bit ? 2 : 0)];
        c = cmul(c, f);
      }
      v[0][0] = c;
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int mo = gpass->init_mat[st0.reg_glob[j]];
        const float2 f0 = mo < 0 ? make_float2(1.f, 0.f) : msm[mo - mat_begin];
        const float2 f1 = mo < 0 ? make_float2(0.f, 0.f) : msm[mo - mat_begin + 2];
#pragma unroll
        for (int r = 0; r < (1 << j); ++r) {
          v[0][r | (1 << j)] = cmul(v[0][r], f1);
          v[0][r] = cmul(v[0][r], f0);
        }
      }
      if constexpr (ADJ) {
#pragma unroll
        for (int r = 0; r < NR; ++r) v[1][r] = make_float2(0.f, 0.f);
      }
    }
  }

  // ---- stages ----
  for (int s = 0; s < st_cnt; ++s) {
    const QfStage& st = sst[s];
    if (s != 0) remap<R, TB, NA>(v, tile, sst[s - 1], st, t);
    const uint32_t gt = base | thread_glob<TB>(st, t);
    const int ob = st.op_begin - op_begin, oe = st.op_end - op_begin;
    for (int k = ob; k < oe; ++k) {
      const QfOp& op = sop[k];  // ADJ programs are emitted in backward execution order
      const int kind = op.kind;
      if (kind == QF_OP_DENSE1) {
        float2 u00, u01, u10, u11;
        load_u2(msm + (op.mat - mat_begin), ADJ, u00, u01, u10, u11);
        const int cls = op.cls;
        if constexpr (ADJ) {
          if (op.slot >= 0) {
            const float2* g = reinterpret_cast<const float2*>(P.genmats) + op.gen;
            const int gk = op.gkind;
            float gacc = 0.f;
            dispatch1<R>(op.s0, [&]<int J>() {
              if (gk == 1) gacc = gradp<J, NR, 1>(v[0], v[1]);
              else if (gk == 2) gacc = gradp<J, NR, 2>(v[0], v[1]);
              else if (gk == 3) gacc = gradp<J, NR, 3>(v[0], v[1]);
              else gacc = grad1<J, NR>(v[0], v[1], g);
            });
            if (gk != 0) gacc *= g[4].x;
            const double gs = warp_sum_d((double)gacc);
            if ((t & 31) == 0) ssm[(op.slot - slot_begin) * NW + (t >> 5)] += gs;
          }
        }
        dispatch1<R>(op.s0, [&]<int J>() {
#pragma unroll
          for (int q = 0; q < NA; ++q) {
            if (cls == 1) apply1<J, NR, 1>(v[q], u00, u01, u10, u11);
            else if (cls == 2) apply1<J, NR, 2>(v[q], u00, u01, u10, u11);
            else apply1<J, NR, 0>(v[q], u00, u01, u10, u11);
          }
        });
      } else if (kind == QF_OP_DENSE2) {
        const float2* u = msm + (op.mat - mat_begin);
        if constexpr (ADJ) {
          if (op.slot >= 0) {
            const float2* g = reinterpret_cast<const float2*>(P.genmats) + op.gen;
            float gacc = 0.f;
            dispatch2<R>(op.s0, op.s1, [&]<int J0, int J1>() { gacc = grad2<J0, J1, NR>(v[0], v[1], g); });
            const double gs = warp_sum_d((double)gacc);
            if ((t & 31) == 0) ssm[(op.slot - slot_begin) * NW + (t >> 5)] += gs;
          }
          dispatch2<R>(op.s0, op.s1, [&]<int J0, int J1>() {
            apply2<J0, J1, NR>(v[0], u, true);
            apply2<J0, J1, NR>(v[1], u, true);
          });
        } else {
          dispatch2<R>(op.s0, op.s1, [&]<int J0, int J1>() { apply2<J0, J1, NR>(v[0], u, false); });
        }
      } else if (kind == QF_OP_DIAG) {
        const int32_t* grp = sgr + (op.grp - grp_begin);
        if constexpr (ADJ) {
          if (op.slot >= 0) {
            float w[NR];
#pragma unroll
            for (int r = 0; r < NR; ++r) w[r] = im_conj_mul(v[1][r], v[0][r]);
            wht<R, float>(w);
            float W[NR];
            subset_accumulate<R, float>(W, grp, stm, gt, [&](uint2, int kk) { return stw[kk]; });
            float acc = 0.f;
#pragma unroll
            for (int r = 0; r < NR; ++r) acc = fmaf(W[r], w[r], acc);
            const double as = warp_sum_d((double)acc);
            if ((t & 31) == 0) ssm[(op.slot - slot_begin) * NW + (t >> 5)] += as;
          }
        }
        uint32_t A[NR];
        subset_accumulate<R, uint32_t>(A, grp, stm, gt, [&](uint2 tm, int) { return tm.y; });
        wht<R, uint32_t>(A);
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          const float2 ph = phase_turns((int32_t)A[r], ADJ);
#pragma unroll
          for (int q = 0; q < NA; ++q) v[q][r] = cmul(v[q][r], ph);
        }
      } else if (kind == QF_OP_OBS) {
        const int32_t* grp = sgr + (op.grp - grp_begin);
        float A[NR];
        subset_accumulate<R, float>(A, grp, stm, gt, [&](uint2 tm, int) { return __int_as_float((int)tm.y); });
        wht<R, float>(A);
        float e = 0.f;
#pragma unroll
        for (int r = 0; r < NR; ++r) e = fmaf(A[r], fmaf(v[0][r].x, v[0][r].x, v[0][r].y * v[0][r].y), e);
        if constexpr (ADJ) {
#pragma unroll
          for (int r = 0; r < NR; ++r) v[1][r] = make_float2(A[r] * v[0][r].x, A[r] * v[0][r].y);
        }
        if (op.slot >= 0) {
          const double es = warp_sum_d((double)e);
          if ((t & 31) == 0) ssm[(op.slot - slot_begin) * NW + (t >> 5)] += es;
        }
      }
    }
  }

  // ---- store (last stage mapping; lanes on qubits 0..4) ----
  if (store) {
    const QfStage& st = sst[st_cnt - 1];
    const uint32_t gt = base | thread_glob<TB>(st, t);
    uint32_t rg[R];
#pragma unroll
    for (int j = 0; j < R; ++j) rg[j] = 1u << st.reg_glob[j];
    gray_walk<R>(gt, rg, [&](auto r, uint32_t g) {
      constexpr int ri = decltype(r)::value;
      psi_row[g] = v[0][ri];
      if constexpr (ADJ) lam_row[g] = v[1][ri];
    });
  }

  if (slot_cnt > 0) {
    __syncthreads();
    const int tiles = 1 << tiles_log2;
    for (int i = t; i < slot_cnt; i += NT) {
      double acc = 0.0;
      for (int w = 0; w < NW; ++w) acc += ssm[i * NW + w];
      a.partials[((size_t)row * P.n_slots + slot_begin + i) * tiles + o] = acc;
    }
  }
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------

template <int L, int R, bool ADJ>
static int launch_pass(const PassArgs& a, const QfPass& hp, cudaStream_t stream) {
  constexpr int NT = 1 << (L - R);
  constexpr int NA = ADJ ? 2 : 1;
  const size_t terms = (size_t)(hp.term_end - hp.term_begin);
  size_t smem = (size_t)NA * (1u << L) * sizeof(float2) + (size_t)(hp.stage_end - hp.stage_begin) * sizeof(QfStage) +
                (size_t)(hp.op_end - hp.op_begin) * sizeof(QfOp) + (size_t)(hp.slot_end - hp.slot_begin) * 8 * (NT / 32) +
                (size_t)(hp.mat_end - hp.mat_begin) * sizeof(float2) + terms * 8 + (ADJ ? terms * 4 : 0) +
                (size_t)(hp.grp_end - hp.grp_begin) * 4;
  // the attribute is per device context: set it on every launch (cheap) instead of once per process
  cudaFuncSetAttribute(pass_kernel<L, R, ADJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (smem > 200 * 1024) {
    set_error("pass %d needs %zu bytes of shared memory", a.pass, smem);
    return 3;
  }
  const unsigned grid = (unsigned)a.rows << a.tiles_log2;
  pass_kernel<L, R, ADJ><<<grid, NT, smem, stream>>>(a);
  return 0;
}

int run_pass(const PassArgs& a, const QfPass& hp, bool adj, cudaStream_t stream) {
  if (hp.relabelled) {  // permuted stores exist only in the plan-specialised kernels (jit.py)
    set_error("pass %d stores a relabelled tile: run it with the plan-specialised kernels", a.pass);
    return 2;
  }
  const int L = a.prog.L, R = a.prog.R;
  if (!adj && R == 5) {
    switch (L) {
      case 10: return launch_pass<10, 5, false>(a, hp, stream);
      case 11: return launch_pass<11, 5, false>(a, hp, stream);
      case 12: return launch_pass<12, 5, false>(a, hp, stream);
      case 13: return launch_pass<13, 5, false>(a, hp, stream);
    }
  } else if (!adj && R == 4) {
    switch (L) {
      case 10: return launch_pass<10, 4, false>(a, hp, stream);
      case 11: return launch_pass<11, 4, false>(a, hp, stream);
      case 12: return launch_pass<12, 4, false>(a, hp, stream);
    }
  } else if (adj && R == 4) {
    switch (L) {
      case 10: return launch_pass<10, 4, true>(a, hp, stream);
      case 11: return launch_pass<11, 4, true>(a, hp, stream);
      case 12: return launch_pass<12, 4, true>(a, hp, stream);
    }
  }
  set_error("unsupported tile geometry L=%d R=%d adj=%d", L, R, (int)adj);
  return 2;
}

}  // namespace qf
