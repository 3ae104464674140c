// Crossbar microbenchmark: shared-memory 64-bit loads vs 32-bit warp shuffles on one B200.
// Question it answers: can warp shuffles move amplitudes between the threads of
// a tile faster than the shared-memory exchange the pass kernels use?  Each variant moves the
// same number of bytes per thread; the kernel reports bytes per clock per SM.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/micro/xbar_bench.cu -o /tmp/xbar && /tmp/xbar
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITER = 4096;

__global__ void lds64_kernel(float* out, int salt) {
  __shared__ float2 sm[4096];
  const unsigned t = threadIdx.x;
  for (int i = t; i < 4096; i += blockDim.x) sm[i] = make_float2(i * 1e-3f, salt);
  __syncthreads();
  float2 acc[8] = {};
  unsigned idx = t;
#pragma unroll 1
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float2 v = sm[(idx + k * 128u) & 4095u];  // conflict-free 64-bit accesses
      acc[k].x += v.x;
      acc[k].y += v.y;
    }
    idx += 1024u;
  }
  float s = 0.f;
  for (int k = 0; k < 8; ++k) s += acc[k].x + acc[k].y;
  if (s == 12345.f) out[blockIdx.x] = s;
}

__global__ void shfl_kernel(float* out, int salt) {
  const unsigned t = threadIdx.x;
  float2 v[8];
  for (int k = 0; k < 8; ++k) v[k] = make_float2(t * 1e-3f + k, salt);
  float2 acc[8] = {};
#pragma unroll 1
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {  // one float2 = two SHFL.BFLY per amplitude
      const float x = __shfl_xor_sync(0xffffffffu, v[k].x, 1 << (k % 5));
      const float y = __shfl_xor_sync(0xffffffffu, v[k].y, 1 << (k % 5));
      acc[k].x += x;
      acc[k].y += y;
      v[k].x += 1e-7f;
    }
  }
  float s = 0.f;
  for (int k = 0; k < 8; ++k) s += acc[k].x + acc[k].y;
  if (s == 12345.f) out[blockIdx.x] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 256, blocks = sms * 4;  // 32 warps per SM
  const double bytes = (double)blocks * threads * ITER * 8 * 8;  // 8 amplitudes x 8 bytes per iteration
  for (int variant = 0; variant < 2; ++variant) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (variant == 0) lds64_kernel<<<blocks, threads>>>(out, rep);
      else shfl_kernel<<<blocks, threads>>>(out, rep);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 1) {
        const double per_clk_sm = bytes / (ms * 1e-3) / sms / (clk * 1e3);
        printf("{\"variant\": \"%s\", \"ms\": %.4f, \"bytes_per_clk_per_sm\": %.1f, \"sm_clock_mhz\": %d}\n",
               variant == 0 ? "LDS.64 (exchange read half)" : "SHFL.BFLY x2 per float2", ms, per_clk_sm, clk / 1000);
      }
    }
  }
  return 0;
}
