// C ABI of libqfb200.so: build / reduce / Pauli / sampler kernels and the extern "C"
// entry points declared in include/qfb200.h.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <mutex>
#include <string>

#include "qf_common.cuh"

namespace qf {


static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
}

static int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return 1;
  }
  return 0;
}

// ---------------------------------------------------------------------------
// per-row op matrices / angles (fp64 math, complex64 / int32-turn outputs)
// ---------------------------------------------------------------------------

struct Z {
  double x, y;
};
__device__ __forceinline__ Z zmul(Z a, Z b) { return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; }
__device__ __forceinline__ Z zadd(Z a, Z b) { return {a.x + b.x, a.y + b.y}; }

struct Recipe {
  QfBuildRecipe r;
};


// y = U x for a factor on a d-dim sub-vector: U = V diag(exp(-i v lambda)) V^dagger for a
// generator factor (no d x d matrix is formed), or the fixed matrix (row stride 4).
__device__ __forceinline__ void factor_apply(const QfBuildRecipe& R, int kind, int src, double v, int row, int d,
                                             Z* x) {
  Z y[4];
  if (kind == 0) {
    const double* ev = R.gen_eval + src * 4;
    const Z* V = reinterpret_cast<const Z*>(R.gen_evec) + src * 16;
    Z w[4];
    for (int k = 0; k < d; ++k) {   // w = diag(ph) V^dagger x
      Z acc{0, 0};
      for (int j = 0; j < d; ++j) acc = zadd(acc, zmul(Z{V[j * 4 + k].x, -V[j * 4 + k].y}, x[j]));
      double sn, cs;
      sincos(-v * ev[k], &sn, &cs);
      w[k] = zmul(Z{cs, sn}, acc);
    }
    for (int i = 0; i < d; ++i) {
      Z acc{0, 0};
      for (int k = 0; k < d; ++k) acc = zadd(acc, zmul(V[i * 4 + k], w[k]));
      y[i] = acc;
    }
  } else {
    const Z* F = reinterpret_cast<const Z*>(R.fixed) + ((size_t)(R.fixed_rows > 1 ? row : 0) * R.n_fixed + src) * 16;
    for (int i = 0; i < d; ++i) {
      Z acc{0, 0};
      for (int j = 0; j < d; ++j) acc = zadd(acc, zmul(F[i * 4 + j], x[j]));
      y[i] = acc;
    }
  }
  for (int i = 0; i < d; ++i) x[i] = y[i];
}

// One thread per (row, op, column): column c of the op's product, applying every factor to it
// in turn (D-fold parallel and O(d^2) per factor: no 4 x 4 temporaries in local memory).
__global__ void build_dense_col_kernel(const QfBuildRecipe R, const float* theta, int64_t tstride, int rows,
                                       float2* mats, int n_mat) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int cols = R.max_dim == 2 ? 2 : 4;     // one-qubit-only programs: no idle column threads
  if (id >= (int64_t)rows * R.n_dense * cols) return;
  const int col = (int)(id & (cols - 1));
  const int64_t ro = cols == 2 ? id >> 1 : id >> 2;
  const int row = (int)(ro / R.n_dense), op = (int)(ro % R.n_dense);
  const int D = R.dense_dim[op];
  if (col >= D) return;
  Z m[4];
  for (int i = 0; i < 4; ++i) m[i] = Z{i == col ? 1.0 : 0.0, 0.0};
  for (int f = R.dense_fbeg[op]; f < R.dense_fbeg[op + 1]; ++f) {
    const int kind = R.factor[3 * f], src = R.factor[3 * f + 1], emb = R.factor[3 * f + 2];
    const double v = kind == 0 ? R.gen_coeff[src] * (double)theta[row * tstride + R.gen_sym[src]] + R.gen_const[src]
                               : 0.0;
    if (emb == 4) {                       // one-qubit op
      factor_apply(R, kind, src, v, row, 2, m);
    } else if (emb == 0) {                // two-qubit factor in the op's order
      factor_apply(R, kind, src, v, row, 4, m);
    } else if (emb == 1) {                // two-qubit factor with swapped qubits
      Z x[4] = {m[0], m[2], m[1], m[3]};
      factor_apply(R, kind, src, v, row, 4, x);
      m[0] = x[0]; m[2] = x[1]; m[1] = x[2]; m[3] = x[3];
    } else {                              // 2: F (x) I (msb), 3: I (x) F (lsb)
      for (int a = 0; a < 2; ++a) {
        const int i0 = emb == 2 ? a : 2 * a, i1 = emb == 2 ? a + 2 : 2 * a + 1;
        Z x[2] = {m[i0], m[i1]};
        factor_apply(R, kind, src, v, row, 2, x);
        m[i0] = x[0];
        m[i1] = x[1];
      }
    }
  }
  float2* out = mats + (size_t)row * n_mat + R.dense_mat[op];
  for (int i = 0; i < D; ++i) out[i * D + col] = make_float2((float)m[i].x, (float)m[i].y);
}


__global__ void build_angle_kernel(const QfBuildRecipe R, const float* theta, int64_t tstride, int rows,
                                   int32_t* angles, int n_ang) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)rows * R.n_terms) return;
  const int row = (int)(id / R.n_terms), k = (int)(id % R.n_terms);
  const int kind = R.term_src[2 * k], src = R.term_src[2 * k + 1];
  double ang;
  if (kind == 2) {  // frame x-mask column: filled by frame_walk_kernel
    angles[(size_t)row * n_ang + k] = 0;
    return;
  }
  if (kind == 0) {
    const double v = R.gen_coeff[src] * (double)theta[row * tstride + R.gen_sym[src]] + R.gen_const[src];
    ang = v * R.term_beta[k];
  } else {
    ang = R.term_const[(size_t)(R.const_rows > 1 ? row : 0) * R.n_const + src];
  }
  double turns = ang * 0.15915494309189535;  // 1/(2 pi)
  turns -= rint(turns);                       // [-0.5, 0.5]
  const long long fx = llrint(turns * 4294967296.0);
  angles[(size_t)row * n_ang + k] = (int32_t)(uint32_t)(unsigned long long)fx;
}

// ---------------------------------------------------------------------------
// slot reduction: out[row, col] = sum_{slot in col} sum_tile partials[row, slot, tile]
// ---------------------------------------------------------------------------

__global__ void reduce_slots_kernel(const double* __restrict__ partials, int rows, int n_slots, int tiles,
                                    const int32_t* col_ptr, const int32_t* slot_list, int n_cols,
                                    double* out, int accumulate, const double* __restrict__ slot_scale,
                                    const double* __restrict__ col_offset) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows * n_cols) return;
  const int row = warp / n_cols, col = warp % n_cols;
  double acc = 0.0;
  for (int s = col_ptr[col]; s < col_ptr[col + 1]; ++s) {
    const double* p = partials + ((size_t)row * n_slots + slot_list[s]) * tiles;
    double part = 0.0;
    for (int i = lane; i < tiles; i += 32) part += p[i];
    part = warp_sum_d(part);
    acc += slot_scale ? part * slot_scale[(size_t)row * n_slots + slot_list[s]] : part;
  }
  if (col_offset) acc += col_offset[col];
  if (lane == 0) out[(size_t)row * n_cols + col] = accumulate ? out[(size_t)row * n_cols + col] + acc : acc;
}

// ---------------------------------------------------------------------------
// generic Pauli-sum kernels (non-diagonal observables)
// ---------------------------------------------------------------------------

constexpr int kExpectChunk = 2048;

__global__ void pauli_expect_kernel(const float2* __restrict__ psi, int n, int n_terms, const uint32_t* xm,
                                    const uint32_t* zm, const int32_t* ny, const float* coefs,
                                    int64_t cstride, double* partials, int chunks) {
  extern __shared__ double tacc[];
  const int row = blockIdx.y, chunk = blockIdx.x;
  const float2* p = psi + ((size_t)row << n);
  const int nw = blockDim.x >> 5;  // per-(term, warp) partials summed in warp order: deterministic
  __syncthreads();
  const uint32_t x0 = (uint32_t)chunk * kExpectChunk;
  const uint32_t len = min((uint32_t)kExpectChunk, (uint32_t)1u << n);
  for (int k = 0; k < n_terms; ++k) {
    const uint32_t m = xm[k], z = zm[k];
    float acc = 0.f;
    for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) {
      const uint32_t x = x0 + i;
      const float2 a = p[x], b = p[x ^ m];
      // conj(b) * a
      float re = fmaf(b.x, a.x, b.y * a.y), im = fmaf(b.x, a.y, -b.y * a.x);
      const int q = ny[k] & 3;
      float v = q == 0 ? re : q == 1 ? -im : q == 2 ? -re : im;  // Re(i^q * (re + i im))
      acc += (__popc(x & z) & 1) ? -v : v;
    }
    const double ad = warp_sum_d((double)acc);
    if ((threadIdx.x & 31) == 0) tacc[k * nw + (threadIdx.x >> 5)] = ad;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < n_terms; k += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += tacc[k * nw + w];
    partials[((size_t)row * n_terms + k) * chunks + chunk] = s * (double)coefs[row * cstride + k];
  }
}

__global__ void pauli_apply_kernel(const float2* __restrict__ psi, float2* __restrict__ lam, int n, int n_terms,
                                   const uint32_t* xm, const uint32_t* zm, const int32_t* ny, const float* coefs,
                                   int64_t cstride) {
  const size_t id = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t dim = (size_t)1 << n;
  const int row = blockIdx.y;
  if (id >= dim) return;
  const uint32_t y = (uint32_t)id;
  const float2* p = psi + (size_t)row * dim;
  float2 acc = make_float2(0.f, 0.f);
  for (int k = 0; k < n_terms; ++k) {
    const uint32_t x = y ^ xm[k];
    const float2 a = p[x];
    float c = coefs[row * cstride + k];
    if (__popc(x & zm[k]) & 1) c = -c;
    const int q = ny[k] & 3;  // i^q * a
    float2 t = q == 0 ? a : q == 1 ? make_float2(-a.y, a.x) : q == 2 ? make_float2(-a.x, -a.y) : make_float2(a.y, -a.x);
    acc.x = fmaf(c, t.x, acc.x);
    acc.y = fmaf(c, t.y, acc.y);
  }
  lam[(size_t)row * dim + y] = acc;
}

// ---------------------------------------------------------------------------
// sampler: numpy Generator(Philox).choice(N, shots, p) semantics
// ---------------------------------------------------------------------------

constexpr int kChunk = 1024;  // amplitudes per warp chunk (32 lanes x 32)

__device__ __forceinline__ void philox4x64_10(uint64_t c[4], uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ull;
      k1 += 0xBB67AE8584CAA73Bull;
    }
    const uint64_t lo0 = 0xD2E7470EE14C6C93ull * c[0], hi0 = __umul64hi(0xD2E7470EE14C6C93ull, c[0]);
    const uint64_t lo1 = 0xCA5A826395121157ull * c[2], hi1 = __umul64hi(0xCA5A826395121157ull, c[2]);
    const uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
  }
}

// uniform number s of a fresh numpy Philox stream with key (k0, k1): block s/4 + 1, word s%4
__device__ __forceinline__ double philox_uniform(uint64_t k0, uint64_t k1, uint64_t s) {
  uint64_t c[4] = {s / 4 + 1, 0, 0, 0};
  philox4x64_10(c, k0, k1);
  const uint64_t w = c[s & 3];
  return (double)(w >> 11) * (1.0 / 9007199254740992.0);
}

__device__ __forceinline__ double lane_chunk_sum(const float2* p) {
  double s = 0.0;
#pragma unroll 8
  for (int j = 0; j < 32; ++j) {
    const float2 a = p[j];
    s += (double)a.x * a.x + (double)a.y * a.y;
  }
  return s;
}

__device__ __forceinline__ double warp_incl_scan(double v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

__global__ void chunk_sum_kernel(const float2* __restrict__ psi, int n, int rows, double* chunk_tot) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nchunk = ((int64_t)1 << n) / kChunk;
  if (warp >= rows * nchunk) return;
  const int64_t row = warp / nchunk, c = warp % nchunk;
  const float2* p = psi + (row << n) + c * kChunk + lane * 32;
  const double incl = warp_incl_scan(lane_chunk_sum(p), lane);
  if (lane == 31) chunk_tot[warp] = incl;
}

__global__ void row_scan_kernel(const double* chunk_tot, int64_t nchunk, double* prefix) {
  // prefix[row, 0..nchunk] exclusive scan, deterministic (fixed segmentation)
  __shared__ double seg[1024];
  const int row = blockIdx.x, t = threadIdx.x, T = blockDim.x;
  const double* c = chunk_tot + row * nchunk;
  double* out = prefix + row * (nchunk + 1);
  const int64_t per = (nchunk + T - 1) / T;
  const int64_t b = t * per, e = min(nchunk, b + per);
  double s = 0.0;
  for (int64_t i = b; i < e; ++i) s += c[i];
  seg[t] = s;
  __syncthreads();
  if (t == 0) {
    double run = 0.0;
    for (int i = 0; i < T; ++i) {
      const double x = seg[i];
      seg[i] = run;
      run += x;
    }
  }
  __syncthreads();
  double run = seg[t];
  for (int64_t i = b; i < e; ++i) {
    out[i] = run;
    run += c[i];
  }
  if (e == nchunk && b < e) out[nchunk] = run;
  if (nchunk == 0 && t == 0) out[0] = 0.0;
}

// One warp per (row, key, shot): kper keys per state row (substream(seed, k) for every
// term k of a sampled expectation draws from one CDF), output [rows, kper, shots].
__global__ void draw_kernel(const float2* __restrict__ psi, int n, int rows, int kper, int shots,
                            const uint64_t* keys, const double* prefix, int64_t* out, int32_t* near) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= (int64_t)rows * kper * shots) return;
  const int krow = (int)(warp / shots);
  const int row = krow / kper;
  const int64_t s = warp % shots;
  const int64_t nchunk = ((int64_t)1 << n) / kChunk;
  const double* pre = prefix + row * (nchunk + 1);
  const double total = pre[nchunk];
  const double u = philox_uniform(keys[2 * krow], keys[2 * krow + 1], (uint64_t)s);
  const double target = u * total;
  // largest chunk c with pre[c] <= target  (c < nchunk)
  int64_t lo = 0, hi = nchunk - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (pre[mid] <= target) lo = mid;
    else hi = mid - 1;
  }
  const int64_t c = lo;
  const float2* p = psi + ((int64_t)row << n) + c * kChunk;
  const double ls = lane_chunk_sum(p + lane * 32);
  const double incl = warp_incl_scan(ls, lane);
  const double base = pre[c];
  const unsigned ball = __ballot_sync(0xffffffffu, base + incl > target);
  int64_t idx;
  double before, after;
  if (ball) {
    const int L = __ffs(ball) - 1;
    double acc = base + __shfl_sync(0xffffffffu, incl - ls, L);
    int j = 31;
    double prev = acc;
    const float2* q = p + L * 32;
    for (int k = 0; k < 32; ++k) {
      const float2 a = q[k];
      prev = acc;
      acc += (double)a.x * a.x + (double)a.y * a.y;
      if (acc > target) { j = k; break; }
    }
    idx = c * kChunk + L * 32 + j;
    before = prev;
    after = acc;
  } else {  // rounding at the chunk edge: clamp to the chunk's last index
    idx = c * kChunk + kChunk - 1;
    before = after = base + __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) {
    out[(int64_t)krow * shots + s] = idx;
    const double tol = 1e-12 * total;
    if (near && (fabs(after - target) < tol || fabs(target - before) < tol)) atomicAdd(near + krow, 1);
  }
}


// ---------------------------------------------------------------------------
// Pauli-frame walk (one thread per row, events in program execution order).
//
// Invariant: true state = sqrt(m) * X^x Z^z * stored state (up to a global phase, which
// cancels in every expectation and in Im<lambda|G|psi> because psi and lambda share it).
//   EV_NX / EV_NY  the op applies A = P^dag U P (U = the built matrix, or U^dag in the
//                  adjoint; P = frame on q).  A = e^{i phi}(c I - i s Q), Q = X or Y, is
//                  written as (c)(I - i t Q) [|c| >= |s|] or (-i s Q)(I + i (c/s) Q), so the
//                  kernel applies I - i tau Q with |tau| <= 1, m *= max(c^2, s^2) and the
//                  second form multiplies the frame by Q.  Gradient slot scale = m * sign,
//                  sign = (-1)^{z_q} (X) or (-1)^{x_q + z_q} (Y) = P^dag Q P / Q.
//   EV_ABS1/ABS2   general dense op: matrix absorbs the frame (M P, or P M in the adjoint
//                  whose kernels apply M^dag), frame bits on its qubits are cleared; its
//                  gradient slot (taken after the apply, frame-free there) scales by m.
//   EV_DIAG/OBS    frame x-mask written to the op's angle column (kernels evaluate the
//                  phase polynomial / observable at index ^ x); slot scale = m.
// ---------------------------------------------------------------------------

__device__ void frame_pauli(int a, int b, Z (&P)[4]) {  // X^a Z^b, row-major 2x2
  // Z^b = diag(1, (-1)^b);  X^a Z^b
  const double zb = b ? -1.0 : 1.0;
  if (!a) {
    P[0] = {1, 0}; P[1] = {0, 0}; P[2] = {0, 0}; P[3] = {zb, 0};
  } else {
    P[0] = {0, 0}; P[1] = {zb, 0}; P[2] = {1, 0}; P[3] = {0, 0};
  }
}

__device__ void frame_walk_row(const int32_t* __restrict__ ev, int n_ev, int adjoint, int row, float2* M,
                               int32_t* angles, int n_ang, double* slot_scale, int n_slots,
                               const QfFrame* frame_in, QfFrame* frame_out, double* pass_m, int n_pass) {
  uint32_t x = 0, z = 0;
  double m = 1.0;
  if (frame_in) {
    x = frame_in[row].x;
    z = frame_in[row].z;
    m = frame_in[row].m;
  }
  // mp: scale of the stored psi.  It equals m unless the adjoint sweep reloads psi from the
  // forward's pass checkpoints (EV_PASS), whose scale the forward walk recorded; slot sums
  // of <lambda|G|psi> then scale by sqrt(m * mp).
  double mp = m;
  for (int e = 0; e < n_ev; ++e) {
    const int32_t* E = ev + (size_t)e * 8;
    const int kind = E[0], q0 = E[1], q1 = E[2], off = E[3], slot = E[4], col = E[5];
    if (kind == 1 || kind == 2) {  // normalised X / Y rotation on q0
      const uint32_t bit = 1u << q0;
      const int ax = (x & bit) ? 1 : 0, bz = (z & bit) ? 1 : 0;
      const int flip = kind == 1 ? bz : (ax ^ bz);
      // merged slot (E[7]: 1 head, 2 member): the head writes the slot scale, every member
      // its scale relative to the head next to tau (the kernel weights its gradient by it)
      float rel = 0.f;
      if (slot >= 0) {
        const double sc = mp == m ? m : sqrt(m * mp);
        const double s_ = flip ? -sc : sc;
        if (E[7] == 2) {
          rel = (float)(s_ / slot_scale[(size_t)row * n_slots + slot]);
        } else {
          slot_scale[(size_t)row * n_slots + slot] = s_;
          rel = 1.f;
        }
      }
      Z u00 = {M[off].x, M[off].y}, u01 = {M[off + 1].x, M[off + 1].y}, u10 = {M[off + 2].x, M[off + 2].y};
      if (adjoint) {  // kernels of the adjoint sweep apply U^dag
        const Z t01 = u01;
        u00.y = -u00.y;
        u01 = {u10.x, -u10.y};
        u10 = {t01.x, -t01.y};
      }
      // U = e^{i phi}(c I - i s Q):  X: u01 = -i e^{i phi} s;  Y: u10 = e^{i phi} s
      const Z sv = kind == 1 ? Z{-u01.y, u01.x} /* i*u01 */ : u10;  // e^{i phi} s
      const double c2 = u00.x * u00.x + u00.y * u00.y, s2 = sv.x * sv.x + sv.y * sv.y;
      double tau;
      if (c2 >= s2) {  // t = s / c (real up to rounding): Re(sv * conj(u00)) / |u00|^2
        tau = (sv.x * u00.x + sv.y * u00.y) / c2;
        if (flip) tau = -tau;
        m *= c2;
        mp *= c2;
      } else {         // tau = -c/s
        double k = (u00.x * sv.x + u00.y * sv.y) / s2;
        if (flip) k = -k;
        tau = -k;
        m *= s2;
        mp *= s2;
        x ^= bit;
        if (kind == 2) z ^= bit;
      }
      M[off] = make_float2((float)tau, rel);
    } else if (kind == 7) {  // normalised two-qubit Pauli-string rotation on (q0 msb, q1 lsb)
      const int code = E[6];
      const int l0 = code & 3, l1 = (code >> 2) & 3;  // 1 X, 2 Y, 3 Z
      const uint32_t b0 = 1u << q0, b1 = 1u << q1;
      // F^dag P F = sign P: X/Y anticommute with a Z frame bit, Y/Z with an X frame bit
      int flip = 0;
      flip ^= ((l0 == 1 || l0 == 2) && (z & b0)) ? 1 : 0;
      flip ^= ((l0 == 2 || l0 == 3) && (x & b0)) ? 1 : 0;
      flip ^= ((l1 == 1 || l1 == 2) && (z & b1)) ? 1 : 0;
      flip ^= ((l1 == 2 || l1 == 3) && (x & b1)) ? 1 : 0;
      if (slot >= 0) {
        const double sc = mp == m ? m : sqrt(m * mp);
        slot_scale[(size_t)row * n_slots + slot] = flip ? -sc : sc;
      }
      // U = e^{i phi}(c I - i s P):  U[0][0] = e^{i phi} c,  U[xm][0] = -i s c0 e^{i phi} with
      // P|00> = c0 |xm>  (c0 = i per Y factor);  the adjoint uses U^dag: (U^dag)[xm][0] = conj(U[0][xm])
      const int xm = ((l0 == 1 || l0 == 2) ? 2 : 0) | ((l1 == 1 || l1 == 2) ? 1 : 0);
      const int ny = (l0 == 2) + (l1 == 2);
      Z u00 = {M[off].x, M[off].y}, uxm;
      if (adjoint) {
        u00.y = -u00.y;
        uxm = {M[off + xm].x, -M[off + xm].y};
      } else {
        uxm = {M[off + xm * 4].x, M[off + xm * 4].y};
      }
      // s e^{i phi} = U[xm][0] * i / c0 = U[xm][0] * i * conj(i^ny)
      Z sv = {-uxm.y, uxm.x};                      // * i
      for (int k = 0; k < ny; ++k) sv = {sv.y, -sv.x};  // * (-i) per Y
      const double c2 = u00.x * u00.x + u00.y * u00.y, s2 = sv.x * sv.x + sv.y * sv.y;
      double tau;
      if (c2 >= s2) {
        tau = (sv.x * u00.x + sv.y * u00.y) / c2;
        if (flip) tau = -tau;
        m *= c2;
        mp *= c2;
      } else {
        double k = (u00.x * sv.x + u00.y * sv.y) / s2;
        if (flip) k = -k;
        tau = -k;
        m *= s2;
        mp *= s2;
        if (l0 == 1 || l0 == 2) x ^= b0;
        if (l0 == 2 || l0 == 3) z ^= b0;
        if (l1 == 1 || l1 == 2) x ^= b1;
        if (l1 == 2 || l1 == 3) z ^= b1;
      }
      M[off] = make_float2((float)tau, 0.f);
    } else if (kind == 3 || kind == 4) {  // absorb the frame into a general dense op
      const int D = kind == 3 ? 2 : 4;
      Z P[16];
      {
        Z A[4], B[4];
        const int qa = q0, qb = kind == 4 ? q1 : -1;
        frame_pauli((x >> qa) & 1, (z >> qa) & 1, A);
        if (D == 2) {
          for (int i = 0; i < 4; ++i) P[i] = A[i];
        } else {
          frame_pauli((x >> qb) & 1, (z >> qb) & 1, B);
          for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j) P[i * 4 + j] = zmul(A[(i >> 1) * 2 + (j >> 1)], B[(i & 1) * 2 + (j & 1)]);
        }
        x &= ~(1u << qa);
        z &= ~(1u << qa);
        if (qb >= 0) {
          x &= ~(1u << qb);
          z &= ~(1u << qb);
        }
      }
      Z U[16], N[16];
      for (int i = 0; i < D * D; ++i) U[i] = {M[off + i].x, M[off + i].y};
      for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j) {
          Z acc{0, 0};
          for (int k = 0; k < D; ++k) {  // forward: U P ; adjoint: P^dag U = P U (real Pauli products)
            const Z p = adjoint ? P[i * D + k] : P[k * D + j];
            if (p.x == 0.0) continue;    // P is a signed permutation: one term per entry
            acc = zadd(acc, adjoint ? Z{p.x * U[k * D + j].x, p.x * U[k * D + j].y}
                                    : Z{p.x * U[i * D + k].x, p.x * U[i * D + k].y});
          }
          N[i * D + j] = acc;
        }
      for (int i = 0; i < D * D; ++i) M[off + i] = make_float2((float)N[i].x, (float)N[i].y);
      if (slot >= 0) {  // after the apply; a fused block's E[7] A slots all scale by m
        const double sc = mp == m ? m : sqrt(m * mp);
        const int cnt = E[7] > 0 ? E[7] : 1;
        for (int j = 0; j < cnt; ++j) slot_scale[(size_t)row * n_slots + slot + j] = sc;
      }
    } else if (kind == 8) {  // pass boundary (checkpointed adjoint): record / reload psi's scale
      if (pass_m) {
        if (!adjoint) pass_m[(size_t)row * n_pass + E[6]] = m;
        else mp = pass_m[(size_t)row * n_pass + E[6]];
      }
    } else if (kind == 5 || kind == 6) {
      angles[(size_t)row * n_ang + col] = (int32_t)x;
      if (slot >= 0) slot_scale[(size_t)row * n_slots + slot] = mp == m ? m : sqrt(m * mp);
    }
  }
  if (frame_out) frame_out[row] = QfFrame{x, z, m};
}


// One CTA per row: the row's matrix slab and the event list are staged in shared memory,
// one thread walks the events (shared-memory latency instead of a global round trip per
// event), the CTA writes the slab back.
__global__ void frame_walk_kernel(const int32_t* __restrict__ ev, int n_ev, int adjoint, int rows,
                                  float2* mats, int n_mat, int32_t* angles, int n_ang, double* slot_scale,
                                  int n_slots, const QfFrame* frame_in, QfFrame* frame_out, double* pass_m,
                                  int n_pass, int n_stage) {
  // n_stage <= n_mat: the slab prefix the events touch (block factor matrices follow it)
  extern __shared__ __align__(16) unsigned char fw_smem[];
  // the event list is the same for every row: read through L1/L2 instead of a per-CTA copy,
  // so the shared-memory footprint (and the rows resident per SM) is set by the slab alone
  float2* Ms = reinterpret_cast<float2*>(fw_smem);
  const int row = blockIdx.x;
  float2* M = mats + (size_t)row * n_mat;
  for (int i = threadIdx.x; i < n_stage; i += blockDim.x) Ms[i] = M[i];
  __syncthreads();
  if (threadIdx.x == 0)
    frame_walk_row(ev, n_ev, adjoint, row, Ms, angles, n_ang, slot_scale, n_slots, frame_in, frame_out, pass_m,
                   n_pass);
  __syncthreads();
  for (int i = threadIdx.x; i < n_stage; i += blockDim.x) M[i] = Ms[i];
}

// Fallback for slabs too large for shared memory: one thread per row on global memory.
__global__ void frame_walk_global_kernel(const int32_t* __restrict__ ev, int n_ev, int adjoint, int rows,
                                         float2* mats, int n_mat, int32_t* angles, int n_ang,
                                         double* slot_scale, int n_slots, const QfFrame* frame_in,
                                         QfFrame* frame_out, double* pass_m, int n_pass) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= rows) return;
  frame_walk_row(ev, n_ev, adjoint, row, mats + (size_t)row * n_mat, angles, n_ang, slot_scale, n_slots,
                 frame_in, frame_out, pass_m, n_pass);
}

}  // namespace qf

using namespace qf;

// ---------------------------------------------------------------------------
// extern "C" entry points
// ---------------------------------------------------------------------------

extern "C" {

const char* qf_last_error(void) { return g_err.c_str(); }

int qf_version(void) { return 1; }

int qf_device_sm_count(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return v;
}

int qf_build_ops(const QfBuildRecipe* recipe, const float* theta, int64_t theta_stride, int rows, float* mats,
                 int n_mat, int32_t* angles, int n_ang, void* stream) {
  if (!recipe || rows < 0) {
    set_error("qf_build_ops: bad arguments");
    return 2;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int T = 128;
  if (recipe->n_dense > 0 && rows > 0) {
    const int64_t tot = (int64_t)rows * recipe->n_dense * (recipe->max_dim == 2 ? 2 : 4);
    build_dense_col_kernel<<<(unsigned)((tot + T - 1) / T), T, 0, s>>>(*recipe, theta, theta_stride, rows,
                                                                       reinterpret_cast<float2*>(mats), n_mat);
    if (check_launch("build_dense_col_kernel")) return 1;
  }
  if (recipe->n_terms > 0 && rows > 0) {
    const int64_t tot = (int64_t)rows * recipe->n_terms;
    build_angle_kernel<<<(unsigned)((tot + T - 1) / T), T, 0, s>>>(*recipe, theta, theta_stride, rows, angles,
                                                                   n_ang);
    if (check_launch("build_angle_kernel")) return 1;
  }
  return 0;
}

static int run_passes_common(const QfProgram* prog, int pb, int pe, float* psi, float* lam, int n, int rows,
                             const float* mats, const int32_t* angles, const float* coefs, double* partials,
                             int tiles_per_row, bool adj, void* stream) {
  if (!prog || n < prog->L || n > 32 || rows < 0) {
    set_error("qf_run_passes: bad arguments (n=%d L=%d)", n, prog ? prog->L : -1);
    return 2;
  }
  if (rows == 0) return 0;
  if ((1 << (n - prog->L)) != tiles_per_row) {
    set_error("tiles_per_row %d does not match n=%d L=%d", tiles_per_row, n, prog->L);
    return 2;
  }
  const QfPass* host_passes = prog->host_passes;
  PassArgs a;
  a.prog = *prog;
  a.psi = reinterpret_cast<float2*>(psi);
  a.lam = reinterpret_cast<float2*>(lam);
  a.mats = reinterpret_cast<const float2*>(mats);
  a.angles = angles;
  a.coefs = coefs;
  a.partials = partials;
  a.n = n;
  a.rows = rows;
  a.tiles_log2 = n - prog->L;
  for (int p = pb; p < pe; ++p) {
    a.pass = p;
    int rc = run_pass(a, host_passes[p], adj, (cudaStream_t)stream);
    if (rc) return rc;
    if (check_launch(adj ? "adjoint pass" : "forward pass")) return 1;
  }
  return 0;
}

int qf_run_passes(const QfProgram* prog, int pass_begin, int pass_end, float* psi, int n, int rows,
                  const float* mats, const int32_t* angles, const float* coefs, double* partials, int tiles_per_row,
                  void* stream) {
  return run_passes_common(prog, pass_begin, pass_end, psi, nullptr, n, rows, mats, angles, coefs, partials,
                           tiles_per_row, false, stream);
}

int qf_adjoint_passes(const QfProgram* prog, int pass_begin, int pass_end, float* psi, float* lam, int n, int rows,
                      const float* mats, const int32_t* angles, const float* coefs, double* partials,
                      int tiles_per_row, void* stream) {
  return run_passes_common(prog, pass_begin, pass_end, psi, lam, n, rows, mats, angles, coefs, partials,
                           tiles_per_row, true, stream);
}

int qf_reduce_slots(const double* partials, int rows, int n_slots, int tiles, const int32_t* col_ptr,
                    const int32_t* slot_list, int n_cols, double* out, int accumulate, void* stream) {
  if (rows == 0 || n_cols == 0) return 0;
  const int64_t warps = (int64_t)rows * n_cols;
  const int T = 256;
  reduce_slots_kernel<<<(unsigned)((warps * 32 + T - 1) / T), T, 0, (cudaStream_t)stream>>>(
      partials, rows, n_slots, tiles, col_ptr, slot_list, n_cols, out, accumulate, nullptr, nullptr);
  return check_launch("reduce_slots_kernel");
}

int qf_reduce_slots_scaled(const double* partials, int rows, int n_slots, int tiles, const int32_t* col_ptr,
                           const int32_t* slot_list, int n_cols, double* out, int accumulate,
                           const double* slot_scale, void* stream) {
  if (rows == 0 || n_cols == 0) return 0;
  const int64_t warps = (int64_t)rows * n_cols;
  const int T = 256;
  reduce_slots_kernel<<<(unsigned)((warps * 32 + T - 1) / T), T, 0, (cudaStream_t)stream>>>(
      partials, rows, n_slots, tiles, col_ptr, slot_list, n_cols, out, accumulate, slot_scale, nullptr);
  return check_launch("reduce_slots_kernel");
}

int qf_reduce_slots_offset(const double* partials, int rows, int n_slots, int tiles, const int32_t* col_ptr,
                           const int32_t* slot_list, int n_cols, double* out, int accumulate,
                           const double* slot_scale, const double* col_offset, void* stream) {
  if (rows == 0 || n_cols == 0) return 0;
  const int64_t warps = (int64_t)rows * n_cols;
  const int T = 256;
  reduce_slots_kernel<<<(unsigned)((warps * 32 + T - 1) / T), T, 0, (cudaStream_t)stream>>>(
      partials, rows, n_slots, tiles, col_ptr, slot_list, n_cols, out, accumulate, slot_scale, col_offset);
  return check_launch("reduce_slots_kernel");
}

int qf_frame_walk_ckpt(const int32_t* events, int n_events, int adjoint, int rows, float* mats, int n_mat,
                       int32_t* angles, int n_ang, double* slot_scale, int n_slots, const QfFrame* frame_in,
                       QfFrame* frame_out, double* pass_m, int n_pass, int n_stage, void* stream) {
  if (rows == 0) return 0;
  if (n_stage <= 0 || n_stage > n_mat) n_stage = n_mat;
  const size_t smem = (size_t)n_stage * sizeof(float2);
  if (smem <= 96 * 1024) {
    // per device context (and cheap): set on every call rather than behind a process-wide flag
    cudaFuncSetAttribute(frame_walk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    frame_walk_kernel<<<rows, 128, smem, (cudaStream_t)stream>>>(
        events, n_events, adjoint, rows, reinterpret_cast<float2*>(mats), n_mat, angles, n_ang, slot_scale,
        n_slots, frame_in, frame_out, pass_m, n_pass, n_stage);
    return check_launch("frame_walk_kernel");
  }
  const int T = 128;
  frame_walk_global_kernel<<<(rows + T - 1) / T, T, 0, (cudaStream_t)stream>>>(
      events, n_events, adjoint, rows, reinterpret_cast<float2*>(mats), n_mat, angles, n_ang, slot_scale, n_slots,
      frame_in, frame_out, pass_m, n_pass);
  return check_launch("frame_walk_global_kernel");
}

// ---------------------------------------------------------------------------
// Block-fused adjoint: gradients of the factors of a fused dense block from the block's
// two-point matrix A = (rho - rho^dag)/2i, rho[j][k] = sum psi_in[j] conj(lam_in[k]) taken at
// the block's input by the adjoint pass (planner.build_program(block=True)).  With W_f the
// product of the block's first f factors (forward order) and G_f = 2 coeff G (non-identity
// part), factor f's value is Im<lam_f|G_f|psi_f> = Tr(W_f^dag G_f W_f A).  A slots per block:
// D diagonal entries A[j][j], then 2 Re A[j][k], 2 Im A[j][k] for j < k.  One thread per
// (row, block), fp64.
// ---------------------------------------------------------------------------
extern "C++" {
template <int D>
__device__ __forceinline__ void block_grads_row(int fb, int fe, int slot0, int row, const int32_t* __restrict__ factors,
                                                const double* __restrict__ gens, const float2* __restrict__ mats,
                                                int n_mat, const double* __restrict__ a, int n_a,
                                                double* __restrict__ out, int n_factors) {
  const double* A = a + (size_t)row * n_a + slot0;
  const float2* M = mats + (size_t)row * n_mat;
  // Tr(W^dag G W A) = Tr(G B) with B = W A W^dag, carried factor by factor: B <- M_f B M_f^dag
  Z Bm[D * D], T[D * D];
  {
    int e = D;
    for (int j = 0; j < D; ++j) {
      Bm[j * D + j] = {A[j], 0.0};
      for (int k = j + 1; k < D; ++k) {
        Bm[j * D + k] = {0.5 * A[e], 0.5 * A[e + 1]};
        Bm[k * D + j] = {0.5 * A[e], -0.5 * A[e + 1]};
        e += 2;
      }
    }
  }
  for (int f = fb; f < fe; ++f) {
    const int moff = factors[f * 3], goff = factors[f * 3 + 1];
    for (int i = 0; i < D; ++i)  // T = M B
      for (int j = 0; j < D; ++j) {
        Z acc{0, 0};
        for (int k = 0; k < D; ++k) {
          const float2 m = M[moff + i * D + k];
          acc = zadd(acc, zmul(Z{m.x, m.y}, Bm[k * D + j]));
        }
        T[i * D + j] = acc;
      }
    for (int i = 0; i < D; ++i)  // B = T M^dag
      for (int j = 0; j < D; ++j) {
        Z acc{0, 0};
        for (int k = 0; k < D; ++k) {
          const float2 m = M[moff + j * D + k];
          acc = zadd(acc, zmul(T[i * D + k], Z{m.x, -m.y}));
        }
        Bm[i * D + j] = acc;
      }
    double val = 0.0;
    if (goff >= 0) {  // Re Tr(G B)
      const double* G = gens + (size_t)goff * 2;
      for (int i = 0; i < D; ++i)
        for (int k = 0; k < D; ++k) {
          const Z g{G[(i * D + k) * 2], G[(i * D + k) * 2 + 1]};
          val += g.x * Bm[k * D + i].x - g.y * Bm[k * D + i].y;
        }
    }
    out[(size_t)row * n_factors + f] = val;
  }
}

__global__ void block_grads_kernel(const int32_t* __restrict__ blocks, int n_blocks,
                                   const int32_t* __restrict__ factors, const double* __restrict__ gens,
                                   const float2* __restrict__ mats, int n_mat, const double* __restrict__ a, int n_a,
                                   double* __restrict__ out, int n_factors, int rows) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (int64_t)rows * n_blocks) return;
  const int row = (int)(tid / n_blocks), b = (int)(tid % n_blocks);
  const int fb = blocks[b * 4], fe = blocks[b * 4 + 1], D = blocks[b * 4 + 2], slot0 = blocks[b * 4 + 3];
  if (D == 4)
    block_grads_row<4>(fb, fe, slot0, row, factors, gens, mats, n_mat, a, n_a, out, n_factors);
  else
    block_grads_row<2>(fb, fe, slot0, row, factors, gens, mats, n_mat, a, n_a, out, n_factors);
}

}  // extern "C++"

int qf_block_grads(const int32_t* blocks, int n_blocks, const int32_t* factors, int n_factors, const double* gens,
                   const float* mats, int n_mat, const double* a, int n_a, double* out, int rows, void* stream) {
  if (rows == 0 || n_blocks == 0) return 0;
  const int64_t n = (int64_t)rows * n_blocks;
  const int T = 128;
  block_grads_kernel<<<(unsigned)((n + T - 1) / T), T, 0, (cudaStream_t)stream>>>(
      blocks, n_blocks, factors, gens, reinterpret_cast<const float2*>(mats), n_mat, a, n_a, out, n_factors, rows);
  return check_launch("block_grads_kernel");
}

int qf_frame_walk(const int32_t* events, int n_events, int adjoint, int rows, float* mats, int n_mat,
                  int32_t* angles, int n_ang, double* slot_scale, int n_slots, const QfFrame* frame_in,
                  QfFrame* frame_out, void* stream) {
  return qf_frame_walk_ckpt(events, n_events, adjoint, rows, mats, n_mat, angles, n_ang, slot_scale, n_slots,
                            frame_in, frame_out, nullptr, 0, 0, stream);
}

int qf_pauli_expect(const float* psi, int n, int rows, int n_terms, const uint32_t* xmask, const uint32_t* zmask,
                    const int32_t* ny, const float* coefs, int64_t coef_stride, double* partials, void* stream) {
  if (rows == 0 || n_terms == 0) return 0;
  if (n > 32) {
    set_error("qf_pauli_expect: n=%d > 32", n);
    return 2;
  }
  const int chunks = (int)(((int64_t)1 << n) + kExpectChunk - 1) / kExpectChunk;
  dim3 grid(chunks, rows);
  pauli_expect_kernel<<<grid, 256, n_terms * 8 * sizeof(double), (cudaStream_t)stream>>>(
      reinterpret_cast<const float2*>(psi), n, n_terms, xmask, zmask, ny, coefs, coef_stride, partials, chunks);
  return check_launch("pauli_expect_kernel");
}

int qf_pauli_apply(const float* psi, float* lam, int n, int rows, int n_terms, const uint32_t* xmask,
                   const uint32_t* zmask, const int32_t* ny, const float* coefs, int64_t coef_stride, void* stream) {
  if (rows == 0) return 0;
  const int64_t dim = (int64_t)1 << n;
  dim3 grid((unsigned)((dim + 255) / 256), rows);
  pauli_apply_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(reinterpret_cast<const float2*>(psi),
                                                              reinterpret_cast<float2*>(lam), n, n_terms, xmask,
                                                              zmask, ny, coefs, coef_stride);
  return check_launch("pauli_apply_kernel");
}

int qf_sample_multi(const float* psi, int n, int rows, int keys_per_row, int shots, const uint64_t* keys,
                    double* scratch, int64_t* out_idx, int32_t* near_boundary, void* stream) {
  if (rows == 0 || shots == 0 || keys_per_row == 0) return 0;
  if (n < 10 || n > 32) {
    set_error("qf_sample: n=%d outside [10, 32] (callers pad small registers)", n);
    return 2;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nchunk = ((int64_t)1 << n) / kChunk;
  double* chunk_tot = scratch;
  double* prefix = scratch + rows * nchunk;
  const float2* p = reinterpret_cast<const float2*>(psi);
  const int64_t warps = rows * nchunk;
  chunk_sum_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(p, n, rows, chunk_tot);
  if (check_launch("chunk_sum_kernel")) return 1;
  row_scan_kernel<<<rows, 1024, 0, s>>>(chunk_tot, nchunk, prefix);
  if (check_launch("row_scan_kernel")) return 1;
  const int64_t dw = (int64_t)rows * keys_per_row * shots;
  draw_kernel<<<(unsigned)((dw * 32 + 255) / 256), 256, 0, s>>>(p, n, rows, keys_per_row, shots, keys, prefix,
                                                               out_idx, near_boundary);
  return check_launch("draw_kernel");
}

// ---------------------------------------------------------------------------
// Relabelled programs (planner.plan_passes_remap) leave qubit q on physical bit pos[q]:
// out[row, j] = in[row, i] with bit pos[q] of i = bit q of j.  Writes are coalesced.
// ---------------------------------------------------------------------------
struct BitMap { int32_t pos[32]; };

__global__ void permute_bits_kernel(const float2* __restrict__ in, float2* __restrict__ out, int n, int64_t total,
                                    BitMap m) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = g >> n;
    const uint64_t j = (uint64_t)g & ((1ull << n) - 1);
    uint64_t i = 0;
#pragma unroll 8
    for (int q = 0; q < n; ++q) i |= ((j >> q) & 1ull) << m.pos[q];
    out[g] = in[(row << n) | (int64_t)i];
  }
}

int qf_permute_bits(const float* in, float* out, int n, int rows, const int32_t* pos, void* stream) {
  if (rows == 0) return 0;
  if (n < 1 || n > 32) {
    set_error("qf_permute_bits: n=%d outside [1, 32]", n);
    return 2;
  }
  BitMap m{};
  for (int q = 0; q < n; ++q) m.pos[q] = pos[q];
  const int64_t total = (int64_t)rows << n;
  const int T = 256;
  const int64_t blocks = std::min<int64_t>((total + T - 1) / T, 148LL * 64);
  permute_bits_kernel<<<(unsigned)blocks, T, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const float2*>(in), reinterpret_cast<float2*>(out), n, total, m);
  return check_launch("permute_bits_kernel");
}

int qf_sample(const float* psi, int n, int rows, int shots, const uint64_t* keys, double* scratch, int64_t* out_idx,
              int32_t* near_boundary, void* stream) {
  return qf_sample_multi(psi, n, rows, 1, shots, keys, scratch, out_idx, near_boundary, stream);
}

}  // extern "C"
