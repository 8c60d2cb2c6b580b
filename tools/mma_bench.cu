// mma_bench.cu -- tcgen05.mma issue/throughput microbenchmark (diagnostics; not part of the library).
// One elected thread issues R back-to-back kind::f16 MMAs (K = 16 each, cycling over a K = 128 tile),
// commits once, waits; cycles per MMA are reported for shapes / operand sources the backward kernel
// could use.  Optional contention: the other warps stream ld.shared.v4 during the MMA stream.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_15922_b200/csrc tools/mma_bench.cu -o /tmp/mma_bench -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#include "ptx.cuh"

using namespace dz::ptx;

constexpr int kReps = 64;  // x 8 K-steps
constexpr int kSmem = 128 * 1024 + 2048;

// MODE 0: SS, A and B K-major; 1: TS (A in TMEM), B K-major; 2: SS, B MN-major; 3: SS, A and B MN-major
template <int M, int N, int MODE, bool CG2>
__global__ void __launch_bounds__(256, 1) mma_kernel(unsigned long long* out, int contend) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw);
  volatile int* stop = reinterpret_cast<volatile int*>(smem + 128 * 1024 + 64);
  uint32_t* tbase = reinterpret_cast<uint32_t*>(smem + 128 * 1024 + 128);
  const uint32_t bar = base + 128 * 1024;
  for (int i = threadIdx.x; i < 128 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    *stop = 0;
    fence_mbar_init();
  }
  if (threadIdx.x < 32) {
    if (CG2) tmem_alloc_2cta<512>(smem_u32(tbase));
    else tmem_alloc<512>(smem_u32(tbase));
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  if (CG2) cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tbase;
  // A: [128 rows][128 K] as two 16 KB SW128 boxes at 0; B: [256 rows][128 K] as two 32 KB boxes at 32 KB
  const uint32_t a0 = base, b0 = base + 32 * 1024;
  constexpr uint32_t idesc = idesc_f16(1, 1, MODE == 3 ? 1 : 0, (MODE >= 2) ? 1 : 0, M, N);
  const bool leader = !CG2 || cluster_ctarank() == 0;
  if (threadIdx.x == 0) {
    unsigned long long t0 = 0, t1 = 0;
    for (int rep = 0; rep < 2; ++rep) {  // rep 0 warms up
      t0 = clock64();
      if (leader) {
        for (int r = 0; r < kReps; ++r) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint64_t ad = MODE == 3 ? sdesc_sw128(a0 + kk * 2048, 16384, 1024)
                                          : sdesc_sw128(a0 + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024);
            const uint64_t bd = MODE >= 2 ? sdesc_sw128(b0 + kk * 2048, 32768, 1024)
                                          : sdesc_sw128(b0 + (kk / 4) * 32768 + (kk % 4) * 32, 16, 1024);
            if (MODE == 1) {
              if (CG2) mma_ts_2cta(tmem, tmem + 256 + kk * 8, bd, idesc, 1);
              else mma_ts(tmem, tmem + 256 + kk * 8, bd, idesc, 1);
            } else {
              if (CG2) mma_ss_2cta(tmem, ad, bd, idesc, 1);
              else mma_ss(tmem, ad, bd, idesc, 1);
            }
          }
        }
        if (CG2) tc_commit_2cta(bar, 3);
        else tc_commit(bar);
      }
      mbar_wait(bar, rep & 1);
      t1 = clock64();
    }
    *stop = 1;
    out[blockIdx.x] = t1 - t0;
  } else if (contend == 2 && threadIdx.x >= 32 && threadIdx.x < 160) {
    // TMEM reads: warps 1..4 (lane quadrants w % 4) load columns [384, 512) repeatedly
    const uint32_t w = threadIdx.x / 32;
    uint32_t acc = 0;
    int it = 0;
    while (!*stop && it < 200000) {
      uint32_t r[32];
      tmem_ld32(tmem + ((w % 4) * 32u << 16) + 384 + (it % 4) * 32, r);
      tmem_wait_ld();
      for (int j = 0; j < 32; ++j) acc ^= r[j];
      ++it;
    }
    if (acc == 0x12345678u) out[blockIdx.x + 4096] = acc;
  } else if (contend == 3 && threadIdx.x >= 32) {
    // shared-memory stores into a region the MMAs do not read
    const uint32_t sbase = base + 96 * 1024;
    int it = 0;
    while (!*stop && it < 2000000) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(sbase + ((threadIdx.x * 16 + j * 4096) & 32767)),
                     "r"(it)
                     : "memory");
      ++it;
    }
  } else if (contend == 1 && threadIdx.x >= 32) {
    uint32_t acc = 0;
    const uint32_t sbase = base + 96 * 1024;  // a region the MMAs do not read
    int it = 0;
    while (!*stop && it < 2000000) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        uint32_t x, y, z, w;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(x), "=r"(y), "=r"(z), "=r"(w)
                     : "r"(sbase + ((threadIdx.x * 16 + j * 4096) & 32767)));
        acc ^= x ^ y ^ z ^ w;
      }
      ++it;
    }
    if (acc == 0x12345678u) out[blockIdx.x + 4096] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (CG2) cluster_sync();
  if (threadIdx.x < 32) {
    if (CG2) tmem_dealloc_2cta<512>(tmem);
    else tmem_dealloc<512>(tmem);
  }
}

// The backward kernel's per-step MMA sequence (attn_bwd_kernel), on a copy of its shared-memory map:
// K' / V [128][128] (two 16 KB boxes each), Q' / dO [64][128] (two 8 KB boxes), P^T / dS^T [128][64].
// VAR bit 0: every MMA bf16 (no fp16 / bf16 switching); bit 1: dQ^T issued as N=64 with K-major A
// (layout not what the math needs: timing only); bit 2: S^T / dP^T only; bit 3: dV / dK / dQ^T only.
__device__ float g_red[148 * 8192];
__device__ float g_src[148 * 8192];
template <int VAR, int RANDOM>
__global__ void __launch_bounds__(352, 1) step_kernel(unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw);
  uint32_t* tbase = reinterpret_cast<uint32_t*>(smem + 160 * 1024 + 128);
  const uint32_t bar = base + 160 * 1024;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u + (uint32_t)RANDOM;
    x ^= x >> 13;
    x *= 0x5bd1e995u;
    x ^= x >> 15;
    // RANDOM: random sign / mantissa / exponent in [2^-3, 2^2) for both halves
    reinterpret_cast<uint32_t*>(smem)[i] = RANDOM ? ((x & 0x83ff83ffu) | (((x >> 10) & 0x00070007u) + 0x000c000cu) << 10)
                                                  : 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
  }
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 8, 1);
    mbar_init(bar + 16, 1);
    mbar_init(bar + 24, 1);
    *reinterpret_cast<volatile int*>(smem + 160 * 1024 + 256) = 0;
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc<512>(smem_u32(tbase));
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tbase;
  constexpr uint32_t kK = 0, kV = 32768, kQ = 65536, kO = 81920, kPT = 98304, kDST = 114688;
  constexpr uint32_t f16 = (VAR & 1) ? 1 : 0;
  constexpr uint32_t iS = idesc_f16(f16, f16, 0, 0, 128, 64), iDP = idesc_f16(1, 1, 0, 0, 128, 64),
                     iDV = idesc_f16(1, 1, 0, 1, 128, 128), iDK = idesc_f16(f16, f16, 0, 1, 128, 128),
                     iDQ = (VAR & 2) ? idesc_f16(f16, f16, 0, 1, 128, 64) : idesc_f16(f16, f16, 1, 1, 128, 64);
  auto dk = [&](uint32_t t, int kk, uint32_t box) { return sdesc_sw128(base + t + (kk / 4) * box + (kk % 4) * 32, 16, 1024); };
  auto dm = [&](uint32_t t, int kk, uint32_t box) { return sdesc_sw128(base + t + kk * 2048, box, 1024); };
  if (threadIdx.x == 0) {
    unsigned long long t0 = 0, t1 = 0;
    constexpr int kSteps = 32;
    for (int rep = 0; rep < 2; ++rep) {
      t0 = clock64();
      for (int i = 0; i < kSteps; ++i) {
        if (!(VAR & 8)) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) mma_ss(tmem + 0, dk(kK, kk, 16384), dk(kQ, kk, 8192), iS, kk > 0);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) mma_ss(tmem + 64, dk(kV, kk, 16384), dk(kO, kk, 8192), iDP, kk > 0);
          if (VAR & 128) tc_commit(bar + 8);
        }
        if (!(VAR & 4)) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) mma_ss(tmem + 256, dk(kPT, kk, 16384), dm(kO, kk, 8192), iDV, 1);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) mma_ss(tmem + 384, dk(kDST, kk, 16384), dm(kQ, kk, 8192), iDK, 1);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_ss(tmem + 128 + (i & 1) * 64, (VAR & 2) ? dk(kK, kk, 16384) : dm(kK, kk, 16384), dm(kDST, kk, 16384), iDQ,
                   kk > 0);
          if (VAR & 128) {
            tc_commit(bar + 16);
            tc_commit(bar + 24);
          }
        }
      }
      tc_commit(bar);
      mbar_wait(bar, rep & 1);
      t1 = clock64();
    }
    const int n = ((VAR & 8) ? 0 : 16) + ((VAR & 4) ? 0 : 16);
    out[blockIdx.x] = t1 - t0;
    out[4096 + blockIdx.x] = (unsigned long long)n * kSteps;
    *reinterpret_cast<volatile int*>(smem + 160 * 1024 + 256) = 1;
  } else if ((VAR & 256) && threadIdx.x >= 32) {
    // shared stores + fence.proxy.async (generic -> async proxy), as the softmax-gradient warps do
    const uint32_t sbase = base + 131072;
    for (int it = 0; it < 20000 && !*reinterpret_cast<volatile int*>(smem + 160 * 1024 + 256); ++it) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(sbase + ((threadIdx.x * 16 + j * 4096) & 16383)),
                     "r"(it)
                     : "memory");
      fence_proxy_async_smem();
      if (VAR & 512) __nanosleep(500);
    }
  } else if ((VAR & 64) && threadIdx.x >= 32) {
    // ALU / MUFU-heavy warps on every sub-partition (the softmax-gradient warps' load)
    float a = threadIdx.x * 1e-3f, c = 0.f;
    for (int it = 0; it < 200000 && !*reinterpret_cast<volatile int*>(smem + 160 * 1024 + 256); ++it) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        a = fmaf(a, 0.999f, 1e-4f);
        c += ex2(a);
      }
    }
    if (c == 1.2345f) out[8000] = 1;
  } else if ((VAR & 16) && threadIdx.x == 32) {
    // bulk loads of 32 KB global -> shared (a region the MMAs do not read), back to back
    const uint32_t lb = base + 160 * 1024 + 512;
    mbar_init(lb, 1);
    fence_mbar_init();
    uint32_t ph = 0;
    for (int it = 0; it < 4000 && !*reinterpret_cast<volatile int*>(smem + 160 * 1024 + 256); ++it) {
      mbar_arrive_expect_tx(lb, 32768);
      bulk_load(base + 131072, g_src + blockIdx.x * 8192, 32768, lb, l2_policy_evict_last());
      mbar_wait(lb, ph);
      ph ^= 1;
    }
  } else if ((VAR & 32) && threadIdx.x == 64) {
    // bulk reduce-add of 32 KB shared -> global fp32, one in flight
    for (int it = 0; it < 4000 && !*reinterpret_cast<volatile int*>(smem + 160 * 1024 + 256); ++it) {
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(g_red + blockIdx.x * 8192),
                   "r"(base + 131072 + 32768), "r"(32768)
                   : "memory");
      bulk_commit_group();
      bulk_wait_read_all();
    }
    bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

// Latency from an idle pipe: issue one group, commit, wait; cycles from the first issue to the wait's
// return, averaged over 32 repetitions.  G = 1: one MMA (M128 N64); 16: S^T / dP^T group; 17: dV / dK /
// dQ^T group; 8: S^T only (8 MMAs into one accumulator).
template <int G, int POLL = 0>
__global__ void __launch_bounds__(320, 1) lat_kernel(unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw);
  uint32_t* tbase = reinterpret_cast<uint32_t*>(smem + 160 * 1024 + 128);
  const uint32_t bar = base + 160 * 1024;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc<512>(smem_u32(tbase));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tbase;
  constexpr uint32_t kK = 0, kV = 32768, kQ = 65536, kO = 81920, kPT = 98304, kDST = 114688;
  constexpr uint32_t iS = idesc_f16(0, 0, 0, 0, 128, 64), iDP = idesc_f16(1, 1, 0, 0, 128, 64),
                     iDV = idesc_f16(1, 1, 0, 1, 128, 128), iDK = idesc_f16(0, 0, 0, 1, 128, 128),
                     iDQ = idesc_f16(0, 0, 1, 1, 128, 64);
  auto dk = [&](uint32_t t, int kk, uint32_t box) { return sdesc_sw128(base + t + (kk / 4) * box + (kk % 4) * 32, 16, 1024); };
  auto dm = [&](uint32_t t, int kk, uint32_t box) { return sdesc_sw128(base + t + kk * 2048, box, 1024); };
  if (threadIdx.x < 32) {
    unsigned long long acc = 0;
    for (int rep = 0; rep < 33; ++rep) {
      const unsigned long long t0 = clock64();
      if (G == 1) {
        mma_ss_warp(tmem, dk(kK, 0, 16384), dk(kQ, 0, 8192), iS, 0);
      } else if (G == 8) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) mma_ss_warp(tmem, dk(kK, kk, 16384), dk(kQ, kk, 8192), iS, kk > 0);
      } else if (G == 16) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) mma_ss_warp(tmem, dk(kK, kk, 16384), dk(kQ, kk, 8192), iS, kk > 0);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) mma_ss_warp(tmem + 64, dk(kV, kk, 16384), dk(kO, kk, 8192), iDP, kk > 0);
      } else {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_ss_warp(tmem + 256, dk(kPT, kk, 16384), dm(kO, kk, 8192), iDV, 1);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_ss_warp(tmem + 384, dk(kDST, kk, 16384), dm(kQ, kk, 8192), iDK, 1);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) mma_ss_warp(tmem + 128, dm(kK, kk, 16384), dm(kDST, kk, 16384), iDQ, kk > 0);
      }
      tc_commit_warp(bar);
      mbar_wait(bar, rep & 1);
      const unsigned long long t1 = clock64();
      if (rep > 0) acc += t1 - t0;
    }
    if (threadIdx.x == 0) out[blockIdx.x] = acc / 32;
  } else if (POLL) {
    // 8 warps wait on the same barrier phases the issuing warp waits on (as the softmax-gradient warps do)
    for (int rep = 0; rep < 33; ++rep) mbar_wait(bar, rep & 1);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}
template <int G, int POLL = 0>
void run_lat(const char* name, unsigned long long* d_out) {
  auto k = lat_kernel<G, POLL>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 170 * 1024);
  k<<<148, POLL ? 288 : 128, 170 * 1024>>>(d_out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%-40s: %s\n", name, cudaGetErrorString(e));
    return;
  }
  unsigned long long h[148];
  cudaMemcpy(h, d_out, sizeof h, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += (double)h[i];
  printf("%-40s: %7.1f clk issue -> commit observed\n", name, s / 148);
}

template <int VAR, int RANDOM = 0>
void run_step(const char* name, unsigned long long* d_out) {
  auto k = step_kernel<VAR, RANDOM>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k<<<148, (VAR & (64 | 256)) ? 352 : 256, 200 * 1024>>>(d_out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%-40s: %s\n", name, cudaGetErrorString(e));
    return;
  }
  unsigned long long h[148], m[1];
  cudaMemcpy(h, d_out, sizeof h, cudaMemcpyDeviceToHost);
  cudaMemcpy(m, d_out + 4096, sizeof m, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += (double)h[i];
  s /= 148;
  printf("%-40s: %8.1f clk/step (32 steps), %6.1f clk/MMA\n", name, s / 32, s / (double)m[0]);
}

// Issue cost: M=128 N=8 MMAs (4-cycle tensor floor), so the issuing thread is the bottleneck.
// STYLE 0: lane 0 of the warp issues (divergent region), descriptors formed per MMA from a loop-varying
// base; 1: the whole warp runs the loop and an elect.sync inside the asm picks the issuing lane;
// 2: as 1 with the elect hoisted: one elect_one() per group, mma_ss under if (leader) inside the loop.
__device__ __forceinline__ void mma_ss_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred E, P;\n\t"
      "elect.sync _|E, 0xffffffff;\n\t"
      "setp.ne.b32 P, %4, 0;\n\t"
      "@E tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, P;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
template <int STYLE>
__global__ void __launch_bounds__(128, 1) issue_kernel(unsigned long long* out, int reps) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw);
  uint32_t* tbase = reinterpret_cast<uint32_t*>(smem + 64 * 1024 + 128);
  const uint32_t bar = base + 64 * 1024;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc<512>(smem_u32(tbase));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tbase;
  constexpr uint32_t idesc = idesc_f16(1, 1, 0, 0, 128, 8);
  unsigned long long t0 = 0, t1 = 0;
  if (threadIdx.x < 32) {
    for (int rep = 0; rep < 2; ++rep) {
      t0 = clock64();
      if (STYLE == 0) {
        if (threadIdx.x == 0) {
          for (int r = 0; r < reps; ++r) {
            const uint32_t a0 = base + (r % 3) * 16384, b0 = base + 49152;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              mma_ss(tmem, sdesc_sw128(a0 + (kk / 4) * 8192 + (kk % 4) * 32, 16, 1024),
                     sdesc_sw128(b0 + (kk / 4) * 1024 + (kk % 4) * 32, 16, 1024), idesc, 1);
          }
          tc_commit(bar);
        }
      } else if (STYLE == 1) {
        for (int r = 0; r < reps; ++r) {
          const uint32_t a0 = base + (r % 3) * 16384, b0 = base + 49152;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_ss_elect(tmem, sdesc_sw128(a0 + (kk / 4) * 8192 + (kk % 4) * 32, 16, 1024),
                         sdesc_sw128(b0 + (kk / 4) * 1024 + (kk % 4) * 32, 16, 1024), idesc, 1);
        }
        if (elect_one()) tc_commit(bar);
        __syncwarp();
      } else {
        const bool leader = elect_one();
        for (int r = 0; r < reps; ++r) {
          const uint32_t a0 = base + (r % 3) * 16384, b0 = base + 49152;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            if (leader)
              mma_ss(tmem, sdesc_sw128(a0 + (kk / 4) * 8192 + (kk % 4) * 32, 16, 1024),
                     sdesc_sw128(b0 + (kk / 4) * 1024 + (kk % 4) * 32, 16, 1024), idesc, 1);
        }
        if (leader) tc_commit(bar);
        __syncwarp();
      }
      mbar_wait(bar, rep & 1);
      t1 = clock64();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}
template <int STYLE>
void run_issue(const char* name, unsigned long long* d_out) {
  auto k = issue_kernel<STYLE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  const int reps = 64;
  k<<<148, 128, 70 * 1024>>>(d_out, reps);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%-40s: %s\n", name, cudaGetErrorString(e));
    return;
  }
  unsigned long long h[148];
  cudaMemcpy(h, d_out, sizeof h, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += (double)h[i];
  printf("%-40s: %6.1f clk per MMA issued (M128 N8)\n", name, s / 148 / (reps * 8));
}

template <int M, int N, int MODE, bool CG2>
void run(const char* name, int grid, int contend, unsigned long long* d_out) {
  auto k = mma_kernel<M, N, MODE, CG2>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = kSmem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG2 ? 2 : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, d_out, contend);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%-34s grid %3d contend %d: %s\n", name, grid, contend, cudaGetErrorString(e));
    return;
  }
  unsigned long long h[296];
  cudaMemcpy(h, d_out, sizeof(unsigned long long) * grid, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < grid; ++i) s += (double)h[i];
  s /= grid;
  const double per = s / (kReps * 8);
  const double flop = 2.0 * M * N * 16 / (CG2 ? 2 : 1);  // per SM
  printf("%-34s grid %3d contend %d: %7.1f clk/MMA  %6.0f FLOP/clk/SM (%.0f%% of 8192)\n", name, grid, contend, per,
         flop / per, 100.0 * flop / per / 8192);
}

int main() {
  unsigned long long* d_out;
  cudaMalloc(&d_out, sizeof(unsigned long long) * 8192);
  run_lat<1>("latency: 1 MMA M128 N64", d_out);
  run_lat<8>("latency: S^T group (8 MMAs)", d_out);
  run_lat<16>("latency: S^T + dP^T group (16 MMAs)", d_out);
  run_lat<17>("latency: dV / dK / dQ^T group (16 MMAs)", d_out);
  run_lat<16, 1>("latency: S^T + dP^T, 8 warps polling", d_out);
  run_issue<0>("issue: lane 0 branch", d_out);
  run_issue<1>("issue: converged warp, elect in asm", d_out);
  run_issue<2>("issue: converged warp, hoisted elect", d_out);
  run_step<0>("step: as in attn_bwd_kernel", d_out);
  run_step<0, 1>("step: as in attn_bwd_kernel, random data", d_out);
  run_step<64>("step: + 10 ALU/MUFU warps", d_out);
  run_step<128>("step: + 3 commits per step", d_out);
  run_step<256>("step: + 10 warps STS + fence.proxy.async", d_out);
  run_step<256 + 512>("step: + STS + fence.proxy.async every 500ns", d_out);
  run_step<16>("step: + bulk loads", d_out);
  run_step<32>("step: + bulk reduce-add", d_out);
  run_step<48>("step: + bulk loads + reduce-add", d_out);
  run_step<4 + 48>("step: S^T / dP^T only + loads + reduce", d_out);
  run_step<4, 1>("step: S^T / dP^T only, random data", d_out);
  run_step<8, 1>("step: dV / dK / dQ^T only, random data", d_out);
  run_step<1>("step: all bf16", d_out);
  run_step<2>("step: dQ^T with K-major A", d_out);
  run_step<4>("step: S^T / dP^T only", d_out);
  run_step<8>("step: dV / dK / dQ^T only", d_out);
  run_step<5>("step: S^T / dP^T only, all bf16", d_out);
  run_step<9>("step: dV / dK / dQ^T only, all bf16", d_out);
  run_step<10>("step: dV / dK / dQ^T only, K-major A", d_out);
  if (getenv("MMA_ALL") == nullptr) return 0;
  for (int contend = 0; contend < 4; ++contend)
    for (int grid : {148}) {
      run<128, 64, 0, false>("cg1 SS  M128 N64 (K,K)", grid, contend, d_out);
      run<128, 128, 0, false>("cg1 SS  M128 N128 (K,K)", grid, contend, d_out);
      run<128, 256, 0, false>("cg1 SS  M128 N256 (K,K)", grid, contend, d_out);
      run<128, 64, 2, false>("cg1 SS  M128 N64 (K,MN)", grid, contend, d_out);
      run<128, 128, 2, false>("cg1 SS  M128 N128 (K,MN)", grid, contend, d_out);
      run<128, 64, 3, false>("cg1 SS  M128 N64 (MN,MN)", grid, contend, d_out);
      run<128, 64, 1, false>("cg1 TS  M128 N64", grid, contend, d_out);
      run<128, 128, 1, false>("cg1 TS  M128 N128", grid, contend, d_out);
      run<128, 256, 1, false>("cg1 TS  M128 N256", grid, contend, d_out);
      run<256, 64, 0, true>("cg2 SS  M256 N64 (K,K)", grid, contend, d_out);
      run<256, 128, 0, true>("cg2 SS  M256 N128 (K,K)", grid, contend, d_out);
      run<256, 256, 0, true>("cg2 SS  M256 N256 (K,K)", grid, contend, d_out);
      run<256, 128, 2, true>("cg2 SS  M256 N128 (K,MN)", grid, contend, d_out);
      run<256, 128, 1, true>("cg2 TS  M256 N128", grid, contend, d_out);
    }
  return 0;
}
