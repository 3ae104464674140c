// Shared device helpers for the B200 state-vector kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/qfb200.h"

namespace qf {

struct PassArgs {
  QfProgram prog;
  float2* psi;
  float2* lam;
  const float2* mats;
  const int32_t* angles;
  const float* coefs;
  double* partials;
  int n;
  int rows;
  int tiles_log2;
  int pass;
};
int run_pass(const PassArgs& a, const QfPass& hp, bool adj, cudaStream_t stream);
void set_error(const char* fmt, ...);

// ---- complex64 arithmetic on Blackwell's packed FP32x2 pipe ----------------
// float2 = (re, im).  Every complex multiply-add is written as two f32x2 FMAs
// (FFMA2 / FMUL2 in SASS, with operand swizzle and scalar broadcast), halving
// the FP instruction count of the naive 8-FMA form.

typedef unsigned long long u64;

__device__ __forceinline__ u64 pk(float lo, float hi) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 upk(u64 r) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(r));
  return make_float2(lo, hi);
}
__device__ __forceinline__ u64 f2mul(u64 a, u64 b) {
  u64 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 f2fma(u64 a, u64 b, u64 c) {
  u64 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// a * x
__device__ __forceinline__ float2 cmul(float2 a, float2 x) {
  u64 d = f2mul(pk(a.x, a.x), pk(x.x, x.y));
  return upk(f2fma(pk(-a.y, a.y), pk(x.y, x.x), d));
}
// a*x + b*y
__device__ __forceinline__ float2 cmad2(float2 a, float2 x, float2 b, float2 y) {
  u64 d = f2mul(pk(a.x, a.x), pk(x.x, x.y));
  d = f2fma(pk(-a.y, a.y), pk(x.y, x.x), d);
  d = f2fma(pk(b.x, b.x), pk(y.x, y.y), d);
  return upk(f2fma(pk(-b.y, b.y), pk(y.y, y.x), d));
}
// acc + a*x
__device__ __forceinline__ float2 cfma(float2 a, float2 x, float2 acc) {
  u64 d = f2fma(pk(a.x, a.x), pk(x.x, x.y), pk(acc.x, acc.y));
  return upk(f2fma(pk(-a.y, a.y), pk(x.y, x.x), d));
}
// [[p, i q], [.., ..]] row: p*x + i*q*y  (p, q real)
__device__ __forceinline__ float2 xrow(float p, float2 x, float q, float2 y) {
  u64 d = f2mul(pk(p, p), pk(x.x, x.y));
  return upk(f2fma(pk(-q, q), pk(y.y, y.x), d));
}
// p*x + q*y  (p, q real)
__device__ __forceinline__ float2 rrow(float p, float2 x, float q, float2 y) {
  u64 d = f2mul(pk(p, p), pk(x.x, x.y));
  return upk(f2fma(pk(q, q), pk(y.x, y.y), d));
}
// Im(conj(a) * b), Re(conj(a) * b)
__device__ __forceinline__ float im_conj_mul(float2 a, float2 b) { return fmaf(a.x, b.y, -a.y * b.x); }
__device__ __forceinline__ float re_conj_mul(float2 a, float2 b) { return fmaf(a.x, b.x, a.y * b.y); }

// exp(-i * 2*pi * a / 2^32) for an int32 "turns" angle (inv: exp(+i ...)).
// Exact integer reduction to the nearest quarter turn, then Taylor polynomials on
// |x| <= pi/4 (sin to x^9, cos to x^8: truncation < 3e-8, i.e. fp32 rounding level).
__device__ __forceinline__ float2 phase_turns(int32_t a, bool inv) {
  const uint32_t ua = (uint32_t)a;
  const uint32_t q = (ua + (1u << 29)) >> 30;
  const int32_t r = (int32_t)(ua - (q << 30));
  const float x = (float)r * 1.4629180792671596e-09f;  // 2*pi / 2^32
  const float x2 = x * x;
  const float s = x * fmaf(x2, fmaf(x2, fmaf(x2, fmaf(x2, 2.7557319e-6f, -1.98412698e-4f), 8.33333333e-3f),
                                    -1.66666667e-1f), 1.f);
  const float c = fmaf(x2, fmaf(x2, fmaf(x2, fmaf(x2, 2.48015873e-5f, -1.38888889e-3f), 4.16666667e-2f), -0.5f),
                       1.f);
  float cs = (q & 1) ? s : c;
  float sn = (q & 1) ? c : s;
  if (q == 1 || q == 2) cs = -cs;
  if (q >= 2) sn = -sn;
  return make_float2(cs, inv ? sn : -sn);
}

template <int N>
struct Ctz {
  static constexpr int value = (N & 1) ? 0 : 1 + Ctz<(N >> 1)>::value;
};
template <>
struct Ctz<0> {
  static constexpr int value = 0;
};

__host__ __device__ constexpr int ctz_c(int x) { return (x & 1) ? 0 : 1 + ctz_c(x >> 1); }
__host__ __device__ constexpr int gray_c(int i) { return i ^ (i >> 1); }

// ---- warp / block helpers ---------------------------------------------------

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// In-place Walsh-Hadamard transform over NR = 2^R register entries:
// out[r] = sum_S in[S] * (-1)^{popc(r & S)}.
template <int R, typename T>
__device__ __forceinline__ void wht(T (&a)[1 << R]) {
#pragma unroll
  for (int j = 0; j < R; ++j) {
#pragma unroll
    for (int r = 0; r < (1 << R); ++r) {
      if (r & (1 << j)) continue;
      T x = a[r], y = a[r | (1 << j)];
      a[r] = x + y;
      a[r | (1 << j)] = x - y;
    }
  }
}

}  // namespace qf
