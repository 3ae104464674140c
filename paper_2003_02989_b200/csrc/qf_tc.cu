// Dense 4-qubit block on the 5th-generation tensor cores (tcgen05 / UMMA, TMEM accumulators)
// with 3xTF32 error compensation -- the prototype of moving FP32-bound dense gate blocks
// (brickwork / QCNN programs at 8 FFMA2 per amplitude per fused 2q block)
// off the FMA pipe.
//
// A 16 x 16 complex unitary U on qubits 0..3 maps each run of 16 amplitudes (a row of the
// state viewed as [rows * 2^(n-4), 16] complex) to U * row.  In real arithmetic with the
// interleaved (re, im) storage of complex64 the row IS a 32-float K vector, so
//     D[m, 2i + c] = sum_{j, d} A[m, 2j + d] * B[2j + d, 2i + c]
// with B[2j][2i] = Re U_ij, B[2j+1][2i] = -Im U_ij, B[2j][2i+1] = Im U_ij, B[2j+1][2i+1] =
// Re U_ij: an M=128, N=32, K=32 GEMM per 128 rows (2048 amplitudes) read and written in place
// of the state's own bytes.  TF32 keeps 10 mantissa bits, so D = A.B_hi + A_lo.B_hi + A.B_lo
// (A_hi = tf32(A) and A_lo = A - A_hi written explicitly, B = B_hi + B_lo split on the host; the
// A_lo.B_lo term is below 2^-22):
// 12 MMAs of m128n32k8 accumulate into one 128-lane x 32-column fp32 TMEM tile.
//
// Per CTA (128 threads, persistent over tiles): each thread stages its row of A and A_lo into
// 128-byte-swizzled K-major shared memory (the canonical UMMA SWIZZLE_128B layout: 16-byte
// chunk c of row r lives at chunk c ^ (r & 7)), one elected thread issues the MMAs and commits
// them to an mbarrier, then every warp reads its 32 TMEM lanes back with tcgen05.ld and stores
// its rows.  B (hi, lo) is staged once per CTA.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "qf_common.cuh"

namespace qf {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// SWIZZLE_128B, K-major: 8-row atoms of 1024 bytes (SBO), LBO 16 bytes (unused), version 1
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);          // start address [0, 14)
  d |= (uint64_t)(1) << 16;                        // leading byte offset [16, 30) (16 B units)
  d |= (uint64_t)(1024 >> 4) << 32;                // stride byte offset [32, 46)
  d |= (uint64_t)1 << 46;                          // version [46, 48) = 1 (sm_100)
  d |= (uint64_t)2 << 61;                          // layout type [61, 64) = SWIZZLE_128B
  return d;
}

// instruction descriptor: D f32, A/B tf32, both K-major, N = 32, M = 128
constexpr uint32_t kIdescTF32 = (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
      :
      : "r"(tmem_d), "l"(da), "l"(db), "r"(kIdescTF32), "r"(accumulate));
}

__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t chunk) {  // byte offset in a SW128 K-major tile
  return row * 128u + ((chunk ^ (row & 7u)) << 4);
}

__global__ void __launch_bounds__(128) dense4_tc_kernel(const float4* __restrict__ in, float4* __restrict__ out,
                                                        int64_t n_tiles, const float4* __restrict__ bmat) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* A = sm;              // 128 rows x 128 B
  unsigned char* Alo = sm + 16384;
  unsigned char* Bh = sm + 32768;     // 32 rows x 128 B (B^T, K-major)
  unsigned char* Bl = sm + 36864;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + 40960);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + 40968);
  const uint32_t t = threadIdx.x, warp = t >> 5, lane = t & 31;

  for (uint32_t i = t; i < 2 * 32 * 8; i += 128) {
    const uint32_t which = i >> 8, n = (i >> 3) & 31, c = i & 7;
    *reinterpret_cast<float4*>((which ? Bl : Bh) + swz(n, c)) = bmat[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tslot;
  uint32_t phase = 0;

  // software pipeline: the next tile's row is loaded into registers while this tile's MMAs run
  // and its accumulator is read back and stored
  // global traffic is coalesced: float4 k of a tile (k = c * 128 + t) is row k / 8, chunk k % 8
  int64_t tile = blockIdx.x;
  float4 nxt[8];
  if (tile < n_tiles) {
    const float4* src = in + tile * 1024;
#pragma unroll
    for (uint32_t c = 0; c < 8; ++c) nxt[c] = src[c * 128 + t];
  }
  for (; tile < n_tiles; tile += gridDim.x) {
    // ---- stage the tile: A_hi = tf32(A) and A_lo = A - A_hi ----
#pragma unroll
    for (uint32_t c = 0; c < 8; ++c) {
      const float4 v = nxt[c];
      const uint32_t k = c * 128 + t, row = k >> 3, ch = k & 7;
      float4 lo;
      lo.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
      lo.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
      lo.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
      lo.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
      // explicit tf32 hi part (hi + lo == v exactly; the MMA's own conversion may round)
      *reinterpret_cast<float4*>(A + swz(row, ch)) = make_float4(v.x - lo.x, v.y - lo.y, v.z - lo.z, v.w - lo.w);
      *reinterpret_cast<float4*>(Alo + swz(row, ch)) = lo;
    }
    asm volatile("fence.proxy.async.shared::cta;");   // generic-proxy stores -> async-proxy (MMA) reads
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (t == 0) {
      const uint32_t a = smem_u32(A), al = smem_u32(Alo), bh = smem_u32(Bh), bl = smem_u32(Bl);
#pragma unroll
      for (uint32_t s = 0; s < 4; ++s)   // K = 32 floats = 4 steps of 8 (32 bytes each)
        umma_tf32(tmem, umma_desc_sw128(a + 32 * s), umma_desc_sw128(bh + 32 * s), s > 0);
#pragma unroll
      for (uint32_t s = 0; s < 4; ++s) umma_tf32(tmem, umma_desc_sw128(al + 32 * s), umma_desc_sw128(bh + 32 * s), 1);
#pragma unroll
      for (uint32_t s = 0; s < 4; ++s) umma_tf32(tmem, umma_desc_sw128(a + 32 * s), umma_desc_sw128(bl + 32 * s), 1);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(mbar)));
    }
    // ---- prefetch the next tile while the tensor cores work (measured: one tile ahead beats two) ----
    const int64_t ntile = tile + gridDim.x;
    if (ntile < n_tiles) {
      const float4* src = in + ntile * 1024;
#pragma unroll
      for (uint32_t c = 0; c < 8; ++c) nxt[c] = src[c * 128 + t];
    }
    // ---- wait for the MMAs, read the accumulator tile back (warp w: TMEM lanes 32w..32w+31) ----
    {
      uint32_t done = 0;
      while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}\n"
            : "=r"(done)
            : "r"(smem_u32(mbar)), "r"(phase));
      }
      phase ^= 1u;
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(tmem + ((warp * 32u) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    // ---- epilogue: row t through the (now free) A buffer, then coalesced stores ----
    (void)lane;
#pragma unroll
    for (uint32_t c = 0; c < 8; ++c)
      *reinterpret_cast<float4*>(A + swz(t, c)) =
          make_float4(__uint_as_float(r[4 * c]), __uint_as_float(r[4 * c + 1]), __uint_as_float(r[4 * c + 2]),
                      __uint_as_float(r[4 * c + 3]));
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();   // every warp has read TMEM and written its rows
    asm volatile("tcgen05.fence::after_thread_sync;");
    float4* dst = out + tile * 1024;
#pragma unroll
    for (uint32_t c = 0; c < 8; ++c) {
      const uint32_t k = c * 128 + t;
      dst[k] = *reinterpret_cast<const float4*>(A + swz(k >> 3, k & 7));
    }
    __syncthreads();   // the A buffer is restaged by the next tile
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

// Tensor-core stages of the tile-pass kernels (planner tc_blocks, jit.py): per (row, block) the
// 16 x 16 product of the stage's dense ops (matrices from the row's slab, applied on register
// slots exactly as apply1m / apply2m do), written as the MMA's B image: [2][32][32] floats, B^T
// rows n = 2i + c of K = 2j + d, tf32 hi then lo.  One warp per (row, block); lane c < 16 carries
// column c of the product in fp64.
__global__ void tc_build_kernel(const float2* __restrict__ mats, int n_mat, int rows, const int32_t* __restrict__ ops,
                                const int32_t* __restrict__ bptr, int n_blocks, float* __restrict__ out) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= (int64_t)rows * n_blocks) return;
  const int row = (int)(warp / n_blocks), blk = (int)(warp % n_blocks);
  const int c = lane & 15;
  double cr[16], ci[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    cr[r] = r == c ? 1.0 : 0.0;
    ci[r] = 0.0;
  }
  const float2* M = mats + (size_t)row * n_mat;
  for (int k = bptr[blk]; k < bptr[blk + 1]; ++k) {
    const int kind = ops[4 * k], moff = ops[4 * k + 1], s0 = ops[4 * k + 2], s1 = ops[4 * k + 3];
    if (kind == 1) {   // 2 x 2 on slot s0
      const float2 m00 = M[moff], m01 = M[moff + 1], m10 = M[moff + 2], m11 = M[moff + 3];
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (r & (1 << s0)) continue;
        const int r1 = r | (1 << s0);
        const double ar = cr[r], ai = ci[r], br = cr[r1], bi = ci[r1];
        cr[r] = m00.x * ar - m00.y * ai + m01.x * br - m01.y * bi;
        ci[r] = m00.x * ai + m00.y * ar + m01.x * bi + m01.y * br;
        cr[r1] = m10.x * ar - m10.y * ai + m11.x * br - m11.y * bi;
        ci[r1] = m10.x * ai + m10.y * ar + m11.x * bi + m11.y * br;
      }
    } else {           // 4 x 4 on slots (s0 msb, s1 lsb)
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (r & ((1 << s0) | (1 << s1))) continue;
        const int idx[4] = {r, r | (1 << s1), r | (1 << s0), r | (1 << s0) | (1 << s1)};
        double xr[4], xi[4];
        for (int j = 0; j < 4; ++j) {
          xr[j] = cr[idx[j]];
          xi[j] = ci[idx[j]];
        }
        for (int i = 0; i < 4; ++i) {
          double yr = 0.0, yi = 0.0;
          for (int j = 0; j < 4; ++j) {
            const float2 m = M[moff + i * 4 + j];
            yr += m.x * xr[j] - m.y * xi[j];
            yi += m.x * xi[j] + m.y * xr[j];
          }
          cr[idx[i]] = yr;
          ci[idx[i]] = yi;
        }
      }
    }
  }
  if (lane >= 16) return;
  // column c of U: U[i][c] = (cr[i], ci[i]);  B^T[n = 2i + cc][k = 2c + d]
  float* O = out + ((size_t)row * n_blocks + blk) * 2048;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const double vals[4] = {cr[i], -ci[i], ci[i], cr[i]};   // (cc, d) = (0,0), (0,1), (1,0), (1,1)
    for (int q = 0; q < 4; ++q) {
      const int n = 2 * i + (q >> 1), k = 2 * c + (q & 1);
      const float f = (float)vals[q];
      const float hi = __uint_as_float(__float_as_uint(f) & 0xFFFFE000u);
      O[n * 32 + k] = hi;
      O[1024 + n * 32 + k] = (float)(vals[q] - (double)hi);
    }
  }
}

}  // namespace qf

extern "C" {

// The B images of a program's tensor-core stages: ops [n_ops, 4] = (kind 1/2, matrix offset,
// slot 0, slot 1) in application order, bptr [n_blocks + 1]; out [rows, n_blocks, 2048] floats.
int qf_tc_build(const float* mats, int n_mat, int rows, const int32_t* ops, const int32_t* bptr, int n_blocks,
                float* out, void* stream) {
  if (rows == 0 || n_blocks == 0) return 0;
  const int64_t warps = (int64_t)rows * n_blocks;
  qf::tc_build_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const float2*>(mats), n_mat, rows, ops, bptr, n_blocks, out);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    qf::set_error("tc_build_kernel launch: %s", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}

// Host: the B operand image of a 16 x 16 complex U (row-major (re, im) doubles), split into
// tf32 hi and lo parts: out[2][32][32] floats, B^T rows (n) of K = 32.
int qf_dense4_tc_prepare(const double* u, float* out) {
  for (int which = 0; which < 2; ++which)
    for (int n = 0; n < 32; ++n)
      for (int k = 0; k < 32; ++k) {
        const int i = n >> 1, c = n & 1, j = k >> 1, d = k & 1;
        const double re = u[2 * (i * 16 + j)], im = u[2 * (i * 16 + j) + 1];
        const double b = (c == 0) ? (d == 0 ? re : -im) : (d == 0 ? im : re);
        const float f = (float)b;
        uint32_t bits;
        memcpy(&bits, &f, 4);
        bits &= 0xFFFFE000u;
        float hi;
        memcpy(&hi, &bits, 4);
        out[which * 1024 + n * 32 + k] = which == 0 ? hi : (float)(b - (double)hi);
      }
  return 0;
}

// out = (U on qubits 0..3) in, for a [rows, 2^n] complex64 state (n >= 4; in != out or ==).
// bmat: device copy of qf_dense4_tc_prepare's image.
int qf_dense4_tc(const float* in, float* out, int n, int rows, const float* bmat, void* stream) {
  if (n < 11 || n > 32) {
    qf::set_error("qf_dense4_tc: n=%d outside [11, 32] (128-row tiles of 16 amplitudes)", n);
    return 2;
  }
  const int64_t n_tiles = ((int64_t)rows << n) >> 11;   // 2048 amplitudes per tile
  const int smem = 40960 + 64;
  cudaFuncSetAttribute(qf::dense4_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qf::dense4_tc_kernel, 128, smem);
  const int64_t cap = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  const int64_t grid = n_tiles < cap ? n_tiles : cap;
  qf::dense4_tc_kernel<<<(unsigned)grid, 128, smem, (cudaStream_t)stream>>>(
      reinterpret_cast<const float4*>(in), reinterpret_cast<float4*>(out), n_tiles,
      reinterpret_cast<const float4*>(bmat));
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    qf::set_error("dense4_tc_kernel launch: %s", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}

}  // extern "C"
