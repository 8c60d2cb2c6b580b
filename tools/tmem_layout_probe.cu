// tmem_layout_probe.cu -- where does a tcgen05.mma.cta_group::2 with M = 128 put D in each CTA's TMEM?
// (diagnostics; not part of the library).  A pair of CTAs; A (64 rows per CTA x K = 16) and B (N = 128,
// 64 rows per CTA) in SW128 K-major shared memory with one non-zero K column, so that one MMA gives
// D[m][n] = A[m][0] * B[n][0]: with B[n][0] = 1 the value names the row m + 1, with A[m][0] = 1 the column
// n + 1.  Every CTA then dumps its 128 lanes x 128 columns.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2602_15922_b200/csrc tools/tmem_layout_probe.cu -o tools/tmem_layout_probe.bin -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "ptx.cuh"

using namespace dz::ptx;

__device__ __forceinline__ uint32_t sw128(int r, int k) { return r * 128 + (((k / 8) ^ (r & 7)) << 4) + (k % 8) * 2; }

// MODE 0: D names the row (B = 1); MODE 1: D names the column (A = 1)
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe(float* out, int mode, int M) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw);
  uint32_t* tbase = reinterpret_cast<uint32_t*>(smem + 32768);
  const uint32_t bar = base + 32768 + 64;
  const uint32_t c = cluster_ctarank();
  // A at 0 (up to 128 rows x 128 B), B at 16 KB (64 rows x 128 B)
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  __syncthreads();
  const int a_rows = M / 2;  // rows of A in this CTA
  if (threadIdx.x < a_rows) {
    const int r = threadIdx.x;
    const float v = mode == 0 ? (float)(c * a_rows + r + 1) : 1.f;
    *reinterpret_cast<__nv_bfloat16*>(smem + sw128(r, 0)) = __float2bfloat16(v);
  }
  if (threadIdx.x < 64) {
    const int r = threadIdx.x;
    const float v = mode == 0 ? 1.f : (float)(c * 64 + r + 1);
    *reinterpret_cast<__nv_bfloat16*>(smem + 16384 + sw128(r, 0)) = __float2bfloat16(v);
  }
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc_2cta<512>(smem_u32(tbase));
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tbase;
  // zero the D columns first (so untouched lanes / columns read 0)
  {
    const uint32_t w = threadIdx.x / 32;
    uint32_t z[32];
    for (int j = 0; j < 32; ++j) z[j] = 0;
    for (int cc = 0; cc < 128; cc += 32) tmem_st32(tmem + ((w * 32u) << 16) + cc, z);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (c == 0 && threadIdx.x == 0) {
    const uint64_t ad = sdesc_sw128(base, 16, 1024), bd = sdesc_sw128(base + 16384, 16, 1024);
    const uint32_t idesc = idesc_f16(1, 1, 0, 0, M, 128);
    mma_ss_2cta(tmem, ad, bd, idesc, 0);
    tc_commit_2cta(bar, 3);
  }
  mbar_wait(bar, 0);
  tc_fence_after();
  {
    const uint32_t w = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int cc = 0; cc < 128; cc += 32) {
      uint32_t r[32];
      tmem_ld32(tmem + ((w * 32u) << 16) + cc, r);
      tmem_wait_ld();
      for (int j = 0; j < 32; ++j) out[((c * 128) + w * 32 + lane) * 128 + cc + j] = __uint_as_float(r[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (threadIdx.x < 32) tmem_dealloc_2cta<512>(tmem);
}

// TS form, M = 128: A from TMEM.  A TMEM word (lane L, column C) holds the bf16 pair (v, v) with
// v = L + 1 (mode 0) or v = 2 C + 1 for the low and 2 C + 2 for the high half (mode 1); B[n][k] = (k == n % 16)
// so D[m][n] = A[m][k = n % 16]: which lane and column the MMA read for row m, K index k.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe_ts(float* out, int mode) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw);
  uint32_t* tbase = reinterpret_cast<uint32_t*>(smem + 32768);
  const uint32_t bar = base + 32768 + 64;
  const uint32_t c = cluster_ctarank();
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  __syncthreads();
  if (threadIdx.x < 64) {  // B rows n = 64 c + r (this CTA's half of N)
    const int r = threadIdx.x, n = 64 * c + r;
    *reinterpret_cast<__nv_bfloat16*>(smem + 16384 + sw128(r, n % 16)) = __float2bfloat16(1.f);
  }
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc_2cta<512>(smem_u32(tbase));
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tbase;
  {
    const uint32_t w = threadIdx.x / 32, lane = threadIdx.x % 32, L = w * 32 + lane;
    uint32_t z[32];
    for (int j = 0; j < 32; ++j) z[j] = 0;
    for (int cc = 0; cc < 128; cc += 32) tmem_st32(tmem + ((w * 32u) << 16) + cc, z);
    uint32_t a[32];
    for (int j = 0; j < 32; ++j) {
      const float lo = mode == 0 ? (float)(L + 1) : (float)(2 * j + 1), hi = mode == 0 ? (float)(L + 1) : (float)(2 * j + 2);
      a[j] = pack_bf16x2(lo, hi);
    }
    tmem_st32(tmem + ((w * 32u) << 16) + 256, a);  // A at columns [256, 288)
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (c == 0 && threadIdx.x == 0) {
    const uint64_t bd = sdesc_sw128(base + 16384, 16, 1024);
    const uint32_t idesc = idesc_f16(1, 1, 0, 0, 128, 128);
    mma_ts_2cta(tmem, tmem + 256, bd, idesc, 0);
    tc_commit_2cta(bar, 3);
  }
  mbar_wait(bar, 0);
  tc_fence_after();
  {
    const uint32_t w = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int cc = 0; cc < 128; cc += 32) {
      uint32_t r[32];
      tmem_ld32(tmem + ((w * 32u) << 16) + cc, r);
      tmem_wait_ld();
      for (int j = 0; j < 32; ++j) out[((c * 128) + w * 32 + lane) * 128 + cc + j] = __uint_as_float(r[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (threadIdx.x < 32) tmem_dealloc_2cta<512>(tmem);
}

int main() {
  {
    float* d;
    cudaMalloc(&d, sizeof(float) * 2 * 128 * 128);
    static float h[2][2][128][128];
    for (int mode = 0; mode < 2; ++mode) {
      cudaMemset(d, 0, sizeof(float) * 2 * 128 * 128);
      cudaFuncSetAttribute(probe_ts, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
      probe_ts<<<2, 128, 40 * 1024>>>(d, mode);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("TS mode %d: %s\n", mode, cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(h[mode], d, sizeof(float) * 2 * 128 * 128, cudaMemcpyDeviceToHost);
    }
    printf("== TS M = 128: D (cta, lane, col) -> A lane read (1-based) / A half-column code (2C+1 lo, 2C+2 hi)\n");
    for (int c = 0; c < 2; ++c)
      for (int lane : {0, 1, 31, 32, 63, 64, 65, 127})
        for (int col : {0, 1, 2, 7, 8, 15, 16, 63}) {
          printf("cta %d lane %3d col %3d : A lane %5.0f  code %5.0f\n", c, lane, col, h[0][c][lane][col], h[1][c][lane][col]);
        }
  }
  if (getenv("PROBE_SS") == nullptr) return 0;
  float* d;
  cudaMalloc(&d, sizeof(float) * 2 * 128 * 128);
  static float h[2][2][128][128];
  for (int M : {128, 256}) {
    for (int mode = 0; mode < 2; ++mode) {
      cudaMemset(d, 0, sizeof(float) * 2 * 128 * 128);
      cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
      probe<<<2, 128, 40 * 1024>>>(d, mode, M);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("M=%d mode %d: %s\n", M, mode, cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(h[mode], d, sizeof(float) * 2 * 128 * 128, cudaMemcpyDeviceToHost);
    }
    printf("== M = %d: (cta, lane, column) -> D[row][n] as row/n (1-based), sampled\n", M);
    for (int c = 0; c < 2; ++c)
      for (int lane : {0, 1, 31, 32, 63, 64, 65, 95, 96, 127})
        for (int col : {0, 1, 63, 64, 65, 127}) {
          const float rv = h[0][c][lane][col], nv = h[1][c][lane][col];
          printf("cta %d lane %3d col %3d : row %5.0f n %5.0f\n", c, lane, col, rv, nv);
        }
  }
  return 0;
}
