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

// ---- complex64 arithmetic (float2 = re, im) --------------------------------

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
// a*x + b*y
__device__ __forceinline__ float2 cmad2(float2 a, float2 x, float2 b, float2 y) {
  float re = fmaf(a.x, x.x, fmaf(-a.y, x.y, fmaf(b.x, y.x, -b.y * y.y)));
  float im = fmaf(a.x, x.y, fmaf(a.y, x.x, fmaf(b.x, y.y, b.y * y.x)));
  return make_float2(re, im);
}
// conj(a)*x + conj(b)*y
__device__ __forceinline__ float2 cjmad2(float2 a, float2 x, float2 b, float2 y) {
  float re = fmaf(a.x, x.x, fmaf(a.y, x.y, fmaf(b.x, y.x, b.y * y.y)));
  float im = fmaf(a.x, x.y, fmaf(-a.y, x.x, fmaf(b.x, y.y, -b.y * y.x)));
  return make_float2(re, im);
}
// Im(conj(a) * b)
__device__ __forceinline__ float im_conj_mul(float2 a, float2 b) { return fmaf(a.x, b.y, -a.y * b.x); }

// exp(-i * 2*pi * a / 2^32) with a an int32 "turns" fixed-point angle; inv flips the sign.
__device__ __forceinline__ float2 phase_turns(int32_t a, bool inv) {
  float s, c;
  sincospif((float)a * 4.656612873077393e-10f, &s, &c);  // a * 2^-31 -> sin(pi x)
  return make_float2(c, inv ? s : -s);
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
