// FFMA2 issue-rate microbenchmark: does the source of the broadcast coefficient (per-thread
// register, kernel parameter / constant bank, immediate) change the FP32x2 FMA throughput?
// The backward tile passes apply rotations as d = tau * swizzle(y) + x with tau uniform per
// CTA (one row, one gate); this measures what each operand form sustains per SM sub-partition.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/ffma2_bench tools/micro/ffma2_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

typedef unsigned long long u64;
__device__ __forceinline__ u64 f2fma(u64 a, u64 b, u64 c) {
  u64 d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ u64 pk(float x, float y) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}

constexpr int NACC = 16, ITER = 2048;

struct Coefs { float c[64]; };

// MODE 0: coefficient in a per-thread register (loaded from global, non-uniform)
// MODE 1: coefficient from the kernel parameter block (uniform, constant bank)
// MODE 2: coefficient from the parameter block indexed by blockIdx (uniform register index)
// MODE 3: compile-time immediate
// MODE 4: two register operands that are accumulators of other chains (x = x + y * z, all R)
template <int MODE>
__global__ void __launch_bounds__(128) bench(const float* __restrict__ g, const Coefs cf, float* out) {
  const int t = threadIdx.x;
  u64 acc[NACC], y[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) {
    acc[i] = pk(g[t + i], g[t + i + 1]);
    y[i] = pk(g[t + 2 * i], g[t + 3 * i]);
  }
  float c;
  if (MODE == 0) c = g[t & 7];
  else if (MODE == 1) c = cf.c[5];
  else if (MODE == 2) c = cf.c[blockIdx.x & 63];
  else c = 0.999f;
  const u64 C = pk(c, -c);
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      if (MODE == 4) acc[i] = f2fma(y[i], y[(i + 1) % NACC], acc[i]);
      else acc[i] = f2fma(C, y[i], acc[i]);
    }
  }
  u64 s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s ^= acc[i];
  if (s == 0x12345) out[t] = 1.f;
}

template <int MODE>
double run(const float* g, float* out, int blocks_per_sm, int n_sm) {
  Coefs cf;
  for (int i = 0; i < 64; ++i) cf.c[i] = 0.5f + i * 1e-3f;
  const int grid = n_sm * blocks_per_sm * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  bench<MODE><<<grid, 128>>>(g, cf, out);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) bench<MODE><<<grid, 128>>>(g, cf, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk_khz;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double warp_instr = 5.0 * grid * 4.0 * ITER * NACC;   // 4 warps per block
  const double cycles = ms * 1e-3 * clk_khz * 1e3;
  return warp_instr / cycles / n_sm / 4.0;                     // FFMA2 per cycle per SMSP
}

int main() {
  int n_sm;
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
  float *g, *out;
  cudaMalloc(&g, 4096 * sizeof(float));
  cudaMemset(g, 0, 4096 * sizeof(float));
  cudaMalloc(&out, 4096 * sizeof(float));
  const char* names[] = {"reg", "param", "param_indexed", "immediate", "all_reg_3src"};
  printf("{");
  for (int bps = 2; bps <= 4; bps += 2) {
    double r[5] = {run<0>(g, out, bps, n_sm), run<1>(g, out, bps, n_sm), run<2>(g, out, bps, n_sm),
                   run<3>(g, out, bps, n_sm), run<4>(g, out, bps, n_sm)};
    for (int m = 0; m < 5; ++m)
      printf("%s\"%s_%dwarps_per_smsp\": %.3f", (bps == 2 && m == 0) ? "" : ", ", names[m], bps, r[m]);
  }
  printf(", \"unit\": \"FFMA2 per cycle per SMSP (at the nominal clock)\"}\n");
  return cudaDeviceSynchronize() != cudaSuccess;
}
