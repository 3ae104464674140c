// Tile-pass kernels: one CTA = one (row, tile) of 2^L amplitudes; each thread keeps
// 2^R amplitudes in registers.  A pass applies a whole run of fused gates whose
// targets lie inside the tile's qubit set Q (|Q| = L, Q contains qubits 0..4 so
// every warp-wide global access is 256 contiguous bytes).  Within a pass the
// planner splits the op list into stages; each stage has a register mapping
// (which tile bits live in registers) and stages are connected by one
// swizzled shared-memory transpose.  Diagonal gates are phase polynomials and
// run in any stage without data movement.
//
// Reference semantics being accelerated: qcflow/sim.py:88-136 (apply_matrix /
// run_ops), sim.py:177-213 (Pauli expectation), gradients.py (the adjoint here
// replaces the parameter-shift loop, oracle = PS).
#include <cuda_runtime.h>
#include <stdint.h>

#include "qf_common.cuh"

namespace qf {


// ---------------------------------------------------------------------------
// dense gates on register slots (compile-time slots, runtime matrices in smem)
// ---------------------------------------------------------------------------

template <int J, int NR>
__device__ __forceinline__ void apply1(float2 (&v)[NR], const float2* __restrict__ u, bool adj) {
  float2 u00 = u[0], u01 = u[1], u10 = u[2], u11 = u[3];
  if (adj) {  // U^dagger
    float2 t = u01;
    u00.y = -u00.y; u11.y = -u11.y;
    u01 = make_float2(u10.x, -u10.y);
    u10 = make_float2(t.x, -t.y);
  }
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    if (r & (1 << J)) continue;
    float2 a = v[r], b = v[r | (1 << J)];
    v[r] = cmad2(u00, a, u01, b);
    v[r | (1 << J)] = cmad2(u10, a, u11, b);
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
    float2 a0 = v[i0], a1 = v[i1], a2 = v[i2], a3 = v[i3];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 o = cmad2(m[i * 4 + 0], a0, m[i * 4 + 1], a1);
      float2 p = cmad2(m[i * 4 + 2], a2, m[i * 4 + 3], a3);
      o.x += p.x; o.y += p.y;
      const int dst = i == 0 ? i0 : i == 1 ? i1 : i == 2 ? i2 : i3;
      v[dst] = o;
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
    float2 t0 = cmad2(g00, p[r], g01, p[r1]);
    float2 t1 = cmad2(g10, p[r], g11, p[r1]);
    acc += im_conj_mul(l[r], t0) + im_conj_mul(l[r1], t1);
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
      float2 u = cmad2(g[i * 4 + 2], p[idx[2]], g[i * 4 + 3], p[idx[3]]);
      t.x += u.x; t.y += u.y;
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
#define QF_P(A, B)                                                         \
  case A * 8 + B:                                                          \
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

template <int R, int TB>
__device__ __forceinline__ uint32_t thread_bits(const QfStage& st, int t, bool phys) {
  uint32_t x = 0;
#pragma unroll
  for (int i = 0; i < TB; ++i)
    if (t & (1 << i)) x ^= phys ? (uint32_t)st.thr_phys[i] : (1u << st.thr_glob[i]);
  return x;
}

// write v (mapping `from`) to smem, read back with mapping `to`.
template <int R, int TB, int NA>
__device__ __forceinline__ void remap(float2 (&v)[NA][1 << R], float2* sm, int tile_elems,
                                      const QfStage& from, const QfStage& to, int t) {
  constexpr int NR = 1 << R;
  __syncthreads();
  {
    const uint32_t base = thread_bits<R, TB>(from, t, true);
    uint32_t ph[R];
#pragma unroll
    for (int j = 0; j < R; ++j) ph[j] = (uint32_t)from.reg_phys[j];
    uint32_t addr = base;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      if (i) addr ^= ph[ctz_c(i)];
#pragma unroll
      for (int a = 0; a < NA; ++a) sm[a * tile_elems + addr] = v[a][gray_c(i)];
    }
  }
  __syncthreads();
  {
    const uint32_t base = thread_bits<R, TB>(to, t, true);
    uint32_t ph[R];
#pragma unroll
    for (int j = 0; j < R; ++j) ph[j] = (uint32_t)to.reg_phys[j];
    uint32_t addr = base;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      if (i) addr ^= ph[ctz_c(i)];
#pragma unroll
      for (int a = 0; a < NA; ++a) v[a][gray_c(i)] = sm[a * tile_elems + addr];
    }
  }
}

// A[S] = sum_{k: subset(k) = S} sign_k(t) * value_k  (subset tables built by the planner)
template <int R, typename T, typename ValFn>
__device__ __forceinline__ void subset_accumulate(T (&A)[1 << R], const QfProgram& P, const QfOp& op,
                                                  uint32_t gt, ValFn&& val) {
  const int32_t* grp = P.grp + op.grp;
#pragma unroll
  for (int S = 0; S < (1 << R); ++S) {
    T acc = T(0);
    const int kb = __ldg(grp + S), ke = __ldg(grp + S + 1);
    for (int k = kb; k < ke; ++k) {
      const uint32_t m = __ldg(P.term_mask + k);
      const T x = val(k);
      acc = (__popc(gt & m) & 1) ? acc - x : acc + x;
    }
    A[S] = acc;
  }
}

// ---------------------------------------------------------------------------
// forward pass kernel
// ---------------------------------------------------------------------------

struct SmemLayout {
  int tile;   // float2 elements of one tile
  int mats;   // float2 elements
  int angs;   // int32
  int coefs;  // float
  int slots;  // float
};

template <int L, int R, bool ADJ>
__global__ void __launch_bounds__(1 << (L - R)) pass_kernel(const PassArgs a) {
  constexpr int NR = 1 << R;
  constexpr int TB = L - R;
  constexpr int NT = 1 << TB;
  constexpr int NA = ADJ ? 2 : 1;  // amplitude arrays (psi, lambda)
  constexpr int TILE = 1 << L;
  extern __shared__ __align__(16) unsigned char smem_raw[];

  const QfProgram& P = a.prog;
  const QfPass& pass = P.passes[a.pass];
  const int t = threadIdx.x;
  const int tiles_log2 = a.tiles_log2;
  const int row = (int)(blockIdx.x >> tiles_log2);
  const uint32_t o = blockIdx.x & ((1u << tiles_log2) - 1u);

  const int mat_begin = pass.mat_begin, mat_cnt = pass.mat_end - pass.mat_begin;
  const int ang_begin = pass.ang_begin, ang_cnt = pass.ang_end - pass.ang_begin;
  const int coef_begin = pass.coef_begin, coef_cnt = pass.coef_end - pass.coef_begin;
  const int slot_begin = pass.slot_begin, slot_cnt = pass.slot_end - pass.slot_begin;

  float2* tile = reinterpret_cast<float2*>(smem_raw);
  float2* msm = tile + NA * TILE;
  int32_t* asm_ = reinterpret_cast<int32_t*>(msm + mat_cnt);
  float* csm = reinterpret_cast<float*>(asm_ + ang_cnt);
  double* ssm = reinterpret_cast<double*>(reinterpret_cast<uintptr_t>(csm + coef_cnt + 1) & ~uintptr_t(7));

  // per-row constants of this pass -> smem
  {
    const float2* src = a.mats + (size_t)row * P.n_mat + mat_begin;
    for (int i = t; i < mat_cnt; i += NT) msm[i] = src[i];
    const int32_t* as = a.angles + (size_t)row * P.n_ang + ang_begin;
    for (int i = t; i < ang_cnt; i += NT) asm_[i] = as[i];
    const float* cs = a.coefs + (size_t)row * P.coef_row_stride + coef_begin;
    for (int i = t; i < coef_cnt; i += NT) csm[i] = cs[i];
    for (int i = t; i < slot_cnt; i += NT) ssm[i] = 0.0;
  }

  // global bits of this tile's outer index
  uint32_t base = 0;
  for (int i = 0; i < pass.n_outer; ++i)
    if (o & (1u << i)) base |= 1u << pass.outer_pos[i];

  const size_t row_elems = (size_t)1 << a.n;
  float2* psi_row = a.psi + (size_t)row * row_elems;
  float2* lam_row = ADJ ? a.lam + (size_t)row * row_elems : nullptr;

  float2 v[NA][NR];
  const QfStage* st0 = P.stages + pass.stage_begin;
  __syncthreads();

  // ---- load / initialise ----
  {
    const uint32_t gt = base | thread_bits<R, TB>(*st0, t, false);
    uint32_t rg[R];
#pragma unroll
    for (int j = 0; j < R; ++j) rg[j] = 1u << st0->reg_glob[j];
    if (pass.init == QF_INIT_LOAD || pass.init == QF_INIT_LOAD_PSI) {
      const bool with_lam = ADJ && pass.init == QF_INIT_LOAD;
      uint32_t g = gt;
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        if (i) g ^= rg[ctz_c(i)];
        v[0][gray_c(i)] = psi_row[g];
        if constexpr (ADJ) v[1][gray_c(i)] = with_lam ? lam_row[g] : make_float2(0.f, 0.f);
      }
    } else if (pass.init == QF_INIT_ZERO) {
      uint32_t g = gt;
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        if (i) g ^= rg[ctz_c(i)];
        v[0][gray_c(i)] = make_float2(g == 0 ? 1.f : 0.f, 0.f);
        if constexpr (ADJ) v[1][gray_c(i)] = make_float2(0.f, 0.f);
      }
    } else {  // product state: amp(x) = prod_q f_q[bit_q(x)], f_q = column 0 of qubit q's leading 2x2
      float2 c = make_float2(1.f, 0.f);
      uint32_t regmask = 0;
#pragma unroll
      for (int j = 0; j < R; ++j) regmask |= rg[j];
      for (int q = 0; q < a.n; ++q) {
        if (regmask & (1u << q)) continue;
        const int mo = pass.init_mat[q];
        const int bit = (gt >> q) & 1;
        float2 f = mo < 0 ? make_float2(bit ? 0.f : 1.f, 0.f) : msm[mo - mat_begin + (bit ? 2 : 0)];
        c = cmul(c, f);
      }
      v[0][0] = c;
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int mo = pass.init_mat[st0->reg_glob[j]];
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
  float gacc = 0.f;  // per-op scalar accumulated over the warp before hitting smem
  const int s_beg = pass.stage_begin, s_end = pass.stage_end;
  for (int s = s_beg; s < s_end; ++s) {
    const QfStage& st = P.stages[s];
    if (s != s_beg) remap<R, TB, NA>(v, tile, TILE, P.stages[s - 1], st, t);
    const uint32_t gt = base | thread_bits<R, TB>(st, t, false);
    const int ob = st.op_begin, oe = st.op_end;
    for (int k = 0; k < oe - ob; ++k) {
      const QfOp op = P.ops[ob + k];  // ADJ programs are emitted in backward execution order
      if (op.kind == QF_OP_DENSE1) {
        const float2* u = msm + (op.mat - mat_begin);
        if constexpr (ADJ) {
          if (op.slot >= 0) {
            const float2* g = reinterpret_cast<const float2*>(P.genmats) + op.gen;
            dispatch1<R>(op.s0, [&]<int J>() { gacc = grad1<J, NR>(v[0], v[1], g); });
            const double gs = warp_sum_d((double)gacc);
            if ((t & 31) == 0) atomicAdd(ssm + (op.slot - slot_begin), gs);
          }
          dispatch1<R>(op.s0, [&]<int J>() {
            apply1<J, NR>(v[0], u, true);
            apply1<J, NR>(v[1], u, true);
          });
        } else {
          dispatch1<R>(op.s0, [&]<int J>() { apply1<J, NR>(v[0], u, false); });
        }
      } else if (op.kind == QF_OP_DENSE2) {
        const float2* u = msm + (op.mat - mat_begin);
        if constexpr (ADJ) {
          if (op.slot >= 0) {
            const float2* g = reinterpret_cast<const float2*>(P.genmats) + op.gen;
            dispatch2<R>(op.s0, op.s1, [&]<int J0, int J1>() { gacc = grad2<J0, J1, NR>(v[0], v[1], g); });
            const double gs = warp_sum_d((double)gacc);
            if ((t & 31) == 0) atomicAdd(ssm + (op.slot - slot_begin), gs);
          }
          dispatch2<R>(op.s0, op.s1, [&]<int J0, int J1>() {
            apply2<J0, J1, NR>(v[0], u, true);
            apply2<J0, J1, NR>(v[1], u, true);
          });
        } else {
          dispatch2<R>(op.s0, op.s1, [&]<int J0, int J1>() { apply2<J0, J1, NR>(v[0], u, false); });
        }
      } else if (op.kind == QF_OP_DIAG) {
        if constexpr (ADJ) {
          if (op.slot >= 0) {
            float w[NR];
#pragma unroll
            for (int r = 0; r < NR; ++r) w[r] = im_conj_mul(v[1][r], v[0][r]);
            wht<R, float>(w);
            float W[NR];
            subset_accumulate<R, float>(W, P, op, gt, [&](int k) { return __ldg(P.term_w + k); });
            float acc = 0.f;
#pragma unroll
            for (int r = 0; r < NR; ++r) acc = fmaf(W[r], w[r], acc);
            const double as = warp_sum_d((double)acc);
            if ((t & 31) == 0) atomicAdd(ssm + (op.slot - slot_begin), as);
          }
        }
        uint32_t A[NR];
        subset_accumulate<R, uint32_t>(A, P, op, gt,
                                       [&](int k) { return (uint32_t)asm_[__ldg(P.term_idx + k) - ang_begin]; });
        wht<R, uint32_t>(A);
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          const float2 ph = phase_turns((int32_t)A[r], ADJ);
#pragma unroll
          for (int q = 0; q < NA; ++q) v[q][r] = cmul(v[q][r], ph);
        }
      } else if (op.kind == QF_OP_OBS) {
        float A[NR];
        subset_accumulate<R, float>(A, P, op, gt, [&](int k) { return csm[__ldg(P.term_idx + k) - coef_begin]; });
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
          if ((t & 31) == 0) atomicAdd(ssm + (op.slot - slot_begin), es);
        }
      }
    }
  }

  // ---- store ----
  if (pass.store) {
    const QfStage& st = P.stages[s_end - 1];
    const uint32_t gt = base | thread_bits<R, TB>(st, t, false);
    uint32_t rg[R];
#pragma unroll
    for (int j = 0; j < R; ++j) rg[j] = 1u << st.reg_glob[j];
    uint32_t g = gt;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      if (i) g ^= rg[ctz_c(i)];
      psi_row[g] = v[0][gray_c(i)];
      if constexpr (ADJ) lam_row[g] = v[1][gray_c(i)];
    }
  }

  if (slot_cnt > 0) {
    __syncthreads();
    const int tiles = 1 << tiles_log2;
    for (int i = t; i < slot_cnt; i += NT)
      a.partials[((size_t)row * P.n_slots + slot_begin + i) * tiles + o] = ssm[i];
  }
}

}  // namespace qf

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------

namespace qf {
template <int L, int R, bool ADJ>
static int launch_pass(const PassArgs& a, const QfPass& hp, cudaStream_t stream) {
  constexpr int NT = 1 << (L - R);
  constexpr int NA = ADJ ? 2 : 1;
  size_t smem = (size_t)NA * (1u << L) * sizeof(float2) +
                (size_t)(hp.mat_end - hp.mat_begin) * sizeof(float2) +
                (size_t)(hp.ang_end - hp.ang_begin) * 4 + (size_t)(hp.coef_end - hp.coef_begin) * 4 +
                (size_t)(hp.slot_end - hp.slot_begin) * 8 + 16;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(pass_kernel<L, R, ADJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  if (smem > 200 * 1024) {
    set_error("pass %d needs %zu bytes of shared memory", a.pass, smem);
    return 3;
  }
  const unsigned grid = (unsigned)a.rows << a.tiles_log2;
  pass_kernel<L, R, ADJ><<<grid, NT, smem, stream>>>(a);
  return 0;
}

int run_pass(const PassArgs& a, const QfPass& hp, bool adj, cudaStream_t stream) {
  const int L = a.prog.L, R = a.prog.R;
  if (!adj && R == 5) {
    switch (L) {
      case 10: return launch_pass<10, 5, false>(a, hp, stream);
      case 11: return launch_pass<11, 5, false>(a, hp, stream);
      case 12: return launch_pass<12, 5, false>(a, hp, stream);
      case 13: return launch_pass<13, 5, false>(a, hp, stream);
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
