// umma2_bench.cu -- cta_group::2 tcgen05.mma throughput (M=256 across a CTA pair).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_15922_b200/csrc tools/umma2_bench.cu -o tools/umma2_bench
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace dz;

__device__ uint8_t g_src[1 << 20];  // L2-resident TMA source (ALU 41..44)

template <int MODE, bool RANDOM, bool TMEM_TRAFFIC, int COMMIT_EVERY = 0, int FENCE = 0, int ALU = 0>  // 0: SS N=128 (QK-like), 1: TS N=128 (PV-like), 2: TS+SS 8+8
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1) bench(long long* cycles, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  __shared__ uint64_t bar, dummy[4], idle;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  const uint32_t rank = ptx::cluster_ctarank();
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) {
    uint32_t x = RANDOM ? (i * 2654435761u + 12345u) : 0u;
    // random fp16/bf16 values of magnitude ~[0.5, 2): sign and mantissa bits random, exponent fixed
    const uint32_t m = RANDOM ? ((x & 0x83FF83FFu) | 0x3C003C00u) : 0u;
    reinterpret_cast<uint4*>(smem_raw + (base - raw))[i] = make_uint4(m, m ^ 0x01230123u, m ^ 0x80008000u, m);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    ptx::mbar_init(ptx::smem_u32(&bar), 1);
    for (int i = 0; i < 4; ++i) ptx::mbar_init(ptx::smem_u32(&dummy[i]), 1);
    ptx::mbar_init(ptx::smem_u32(&idle), 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc_2cta<512>(ptx::smem_u32(&tbase));
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  if (rank == 0 && threadIdx.x == 0) {
    constexpr uint32_t idesc_ss = ptx::idesc_f16(0, 0, 0, 0, 256, 128);
    constexpr uint32_t idesc_ts = ptx::idesc_f16(1, 1, 0, 1, 256, 128);
    const uint32_t a = base, b = base + 32768;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (FENCE & 1) ptx::tc_fence_after();
      if (FENCE & 2) ptx::mbar_wait(ptx::smem_u32(&idle), 1);  // already-complete phase
      if (MODE == 1 || MODE == 2) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          ptx::mma_ts_2cta(tmem + 256, tmem + kk * 8, ptx::sdesc_sw128(b + kk * 2048, 16, 1024), idesc_ts, 1);
      }
      if (MODE == 3 || MODE == 5) {  // half-unit QK: M = 128 per pair (64 rows per CTA)
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t qoff = (kk / 4) * 16384 + (kk % 4) * 32, koff = (kk / 4) * 8192 + (kk % 4) * 32;
          ptx::mma_ss_2cta(tmem + 128, ptx::sdesc_sw128(a + qoff, 16, 1024), ptx::sdesc_sw128(b + koff, 16, 1024),
                           ptx::idesc_f16(0, 0, 0, 0, 128, 128), 1);
        }
      }
      if (MODE == 4 || MODE == 5) {  // half-unit PV: P (K-major, 64 rows per CTA) x V (MN-major), M = 128
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          ptx::mma_ss_2cta(tmem + 256, ptx::sdesc_sw128(a + (kk / 4) * 8192 + (kk % 4) * 32, 16, 1024),
                           ptx::sdesc_sw128(b + kk * 2048, 16, 1024), ptx::idesc_f16(1, 1, 0, 1, 128, 128), 1);
      }
      if (MODE == 0 || MODE == 2) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t qoff = (kk / 4) * 16384 + (kk % 4) * 32, koff = (kk / 4) * 8192 + (kk % 4) * 32;
          ptx::mma_ss_2cta(tmem + 128, ptx::sdesc_sw128(a + qoff, 16, 1024), ptx::sdesc_sw128(b + koff, 16, 1024),
                           idesc_ss, 1);
        }
      }
      if (COMMIT_EVERY > 0 && (it % COMMIT_EVERY) == 0) ptx::tc_commit_2cta(ptx::smem_u32(&dummy[it & 3]), 0x3);
    }
    ptx::tc_commit_2cta(ptx::smem_u32(&bar), 0x3);
    ptx::mbar_wait(ptx::smem_u32(&bar), 0);
    long long t1 = clock64();
    cycles[blockIdx.x / 2] = t1 - t0;
    *(volatile uint32_t*)&tbase = 0xFFFFFFFFu;  // stop local TMEM traffic
  }
  if (rank == 1 && threadIdx.x == 0) {
    ptx::mbar_wait(ptx::smem_u32(&bar), 0);
    *(volatile uint32_t*)&tbase = 0xFFFFFFFFu;
  }
  // ALU 2: math on all 4 SMSPs; ALU 20: the same math but never on SMSP 0 (the MMA issuer's)
  if ((ALU == 1 || ALU == 2 || ALU == 20) && warp >= 4 && !(ALU == 20 && warp % 4 == 0)) {
    float a[16];
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
    uint32_t acc = 0;
    for (int k = 0; *(volatile uint32_t*)&tbase != 0xFFFFFFFFu; ++k) {
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        const uint64_t x = ptx::f2_fma(ptx::f2_pack(a[i], a[i + 1]), ptx::f2_pack(0.5f, 0.5f), ptx::f2_pack(-1.f, -1.f));
        float x0, x1;
        ptx::f2_unpack(x, x0, x1);
        if ((ALU == 2 || ALU == 20) && (i & 2)) {
          const uint64_t p = ptx::f2_exp2_poly(x);
          ptx::f2_unpack(p, x0, x1);
        } else {
          x0 = ptx::ex2(x0);
          x1 = ptx::ex2(x1);
        }
        acc += ptx::pack_bf16x2(x0, x1);
        a[i] = x0 * 0.999f;
        a[i + 1] = x1 * 0.999f;
      }
    }
    if (acc == 0x12345) cycles[100] = acc;
  }
  if (ALU >= 3 && ALU < 30 && warp >= 4) {  // 8 warps of one instruction kind only (which pipes interfere with the MMA?)
    float a[16];
    uint64_t v[8];
    uint32_t u[8];
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
    for (int i = 0; i < 8; ++i) { v[i] = ptx::f2_pack(a[i], a[i + 8]); u[i] = threadIdx.x + i; }
    const uint64_t c2 = ptx::f2_pack(0.999f, 0.999f), d2 = ptx::f2_pack(0.001f, 0.001f);
    for (int k = 0; *(volatile uint32_t*)&tbase != 0xFFFFFFFFu; ++k) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (ALU == 3) a[i] = fmaf(a[i], 0.999f, a[i + 8]);
          if (ALU == 4) v[i] = ptx::f2_fma(v[i], c2, d2);
          if (ALU == 5) u[i] = ptx::pack_bf16x2(__uint_as_float(u[i]), a[i]);
          if (ALU == 6) a[i] = ptx::ex2(a[i]);
          if (ALU == 7) v[i] = ptx::f2_add(v[i], d2);
          if (ALU == 8) u[i] = u[i] * 0x9E3779B1u + 7u;
          if (ALU == 9) v[i] = ptx::f2_exp2_poly<false>(v[i]);
          if (ALU == 10) v[i] = ptx::f2_exp2_poly<true>(v[i]);
          if (ALU == 11) { float x, y; ptx::f2_unpack(v[i], x, y); v[i] = ptx::f2_fma(ptx::f2_pack(ptx::ex2(x), ptx::ex2(y)), c2, d2); }
          if (ALU == 12) a[i] = fmaxf(a[i], a[i + 8]) * 0.999f;
          if (ALU == 13) u[i] = __float_as_uint(a[i]) + (u[i] << 23);
        }
    }
    float sacc = 0;
    for (int i = 0; i < 8; ++i) { float x, y; ptx::f2_unpack(v[i], x, y); sacc += a[i] + x + y + __uint_as_float(u[i]); }
    if (sacc == 1.2345f) cycles[100] = 1;
  }
  if (ALU >= 30 && ALU < 40 && warp >= 4) {  // the K2 exponential block (exp_half<true>): poly share ALU - 30 of 8
    constexpr int kP = ALU - 30;
    float s[64];
    for (int i = 0; i < 64; ++i) s[i] = ((threadIdx.x * 131 + i * 17) % 61) - 30.5f;
    uint32_t x = 0;
    for (int k = 0; *(volatile uint32_t*)&tbase != 0xFFFFFFFFu; ++k) {
      uint64_t acc[4] = {0, 0, 0, 0};
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        uint64_t xx = ptx::f2_pack(s[2 * i], s[2 * i + 1]);
        uint64_t p;
        if ((i % 8) >= 8 - kP) {
          p = ptx::f2_exp2_poly<false>(xx);
        } else {
          float x0, x1;
          ptx::f2_unpack(xx, x0, x1);
          p = ptx::f2_pack(ptx::ex2(x0), ptx::ex2(x1));
        }
        acc[i % 4] = ptx::f2_add(acc[i % 4], p);
        float p0, p1;
        ptx::f2_unpack(p, p0, p1);
        x ^= ptx::pack_bf16x2(p0, p1);
      }
      const uint64_t a = ptx::f2_add(ptx::f2_add(acc[0], acc[1]), ptx::f2_add(acc[2], acc[3]));
      float a0, a1;
      ptx::f2_unpack(a, a0, a1);
      x += __float_as_uint(a0 + a1);
      s[k & 63] = __uint_as_float(__float_as_uint(s[k & 63]) ^ (x & 1));
    }
    if (x == 0x12345) cycles[100] = x;
  }
  if (ALU >= 41 && ALU <= 44 && warp == 5) {  // TMA bulk loads (16 KB each, ALU - 40 in flight) into smem [64K, 96K)
    constexpr int kIn = ALU - 40;
    __shared__ uint64_t tbar[4];
    if ((threadIdx.x % 32) == 0) {
      for (int i = 0; i < 4; ++i) ptx::mbar_init(ptx::smem_u32(&tbar[i]), 1);
      ptx::fence_mbar_init();
    }
    __syncwarp();
    uint32_t k = 0, ph[4] = {0, 0, 0, 0};
    const uint64_t pol = ptx::l2_policy_evict_last();
    while (*(volatile uint32_t*)&tbase != 0xFFFFFFFFu) {
      const int sl = k % kIn;
      if ((threadIdx.x % 32) == 0) {
        if (k >= (uint32_t)kIn) { ptx::mbar_wait(ptx::smem_u32(&tbar[sl]), ph[sl]); ph[sl] ^= 1; }
        ptx::mbar_arrive_expect_tx(ptx::smem_u32(&tbar[sl]), 16384);
        ptx::bulk_load(base + 65536 + (sl % 2) * 16384, g_src + ((k * 16384u) & ((1u << 20) - 1)), 16384,
                       ptx::smem_u32(&tbar[sl]), pol);
      }
      __syncwarp();
      ++k;
    }
    if ((threadIdx.x % 32) == 0 && k > 0) {
      for (int i = 0; i < kIn && i < (int)k; ++i) { const int sl = (k - 1 - i) % kIn; ptx::mbar_wait(ptx::smem_u32(&tbar[sl]), ph[sl]); ph[sl] ^= 1; }
    }
    if ((threadIdx.x % 32) == 0) atomicMax((unsigned long long*)&cycles[101], (unsigned long long)k);
  }
  if (TMEM_TRAFFIC && warp >= 4) {  // 8 warps: softmax-like S loads and P stores
    const uint32_t lanes = (uint32_t)((warp % 4) * 32) << 16;
    uint32_t r[32];
    for (int k = 0; *(volatile uint32_t*)&tbase != 0xFFFFFFFFu; ++k) {
      ptx::tmem_ld32(tmem + lanes + (k & 3) * 32, r);
      ptx::tmem_wait_ld();
      ptx::tmem_st32(tmem + lanes + 128 + ((warp / 4 - 1) * 64) + (k & 1) * 32, r);
      ptx::tmem_wait_st();
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  if (warp == 0) ptx::tmem_dealloc_2cta<512>(tmem);  // tmem captured before tbase was overwritten
}

template <int MODE, bool RANDOM, bool TT, int CE = 0, int FE = 0, int AL = 0>
void run(const char* name, double instr_per_iter) {
  long long* d;
  cudaMalloc(&d, 128 * sizeof(long long));
  cudaMemset(d, 0, 128 * sizeof(long long));
  const int iters = 4096;
  auto k = bench<MODE, RANDOM, TT, CE, FE, AL>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<<<148, 384, 100 * 1024>>>(d, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<148, 384, 100 * 1024>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[74];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 74; ++i) avg += h[i];
  avg /= 74;
  const double instrs = iters * instr_per_iter;
  const double flop = 74.0 * instrs * 2.0 * 256 * 128 * 16;
  long long tma_loads = 0;
  cudaMemcpy(&tma_loads, d + 101, sizeof tma_loads, cudaMemcpyDeviceToHost);
  if (tma_loads) printf("[TMA: %.1f B/clk per CTA] ", tma_loads * 16384.0 / avg);
  printf("%-30s cyc/instr %7.2f (ideal 64)  %8.1f TFLOP/s  err=%s\n", name, avg / instrs, flop / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  if (getenv("ONLY_HALF")) {  // M = 128 pair MMAs (half units), per instruction against M = 256
    run<0, true, false>("2CTA SS M256 N128 random", 8);
    run<3, true, false>("2CTA SS M128 N128 (QK half)", 8);
    run<4, true, false>("2CTA SS M128 N128 (PV half)", 8);
    run<5, true, false>("2CTA QK+PV half", 16);
    run<2, true, false>("2CTA TS+SS M256", 16);
    return 0;
  }
  if (getenv("ONLY_TMA")) {
    run<0, true, false, 1, 0, 41>("SS + TMA 16KB x1 in flight", 8);
    run<0, true, false, 1, 0, 42>("SS + TMA 16KB x2 in flight", 8);
    run<0, true, false, 1, 0, 44>("SS + TMA 16KB x4 in flight", 8);
    run<2, true, false, 1, 0, 42>("TS+SS + TMA 16KB x2", 16);
    run<2, true, false, 1, 0, 44>("TS+SS + TMA 16KB x4", 16);
    run<1, true, false, 1, 0, 44>("TS + TMA 16KB x4", 8);
    return 0;
  }
  if (getenv("ONLY_K2")) {
    run<2, true, false, 1, 0, 30>("TS+SS + 8 warps K2 exp (poly 0/8)", 16);
    run<2, true, false, 1, 0, 31>("TS+SS + 8 warps K2 exp (poly 1/8)", 16);
    run<2, true, false, 1, 0, 32>("TS+SS + 8 warps K2 exp (poly 2/8)", 16);
    run<2, true, false, 1, 0, 33>("TS+SS + 8 warps K2 exp (poly 3/8)", 16);
    run<2, true, false, 1, 0, 34>("TS+SS + 8 warps K2 exp (poly 4/8)", 16);
    run<2, true, false, 1, 0, 9>("TS+SS + 8 warps poly (no clamp)", 16);
    run<2, true, false, 1, 0, 3>("TS+SS + 8 warps FFMA", 16);
    return 0;
  }
  if (getenv("ONLY_ALU")) {
    run<2, true, false, 1, 0, 2>("TS+SS + 8 warps MUFU+poly math", 16);
    run<2, true, false, 1, 0, 20>("TS+SS + 6 warps MUFU+poly, SMSP0 free", 16);
    run<2, true, false, 1, 0, 9>("TS+SS + 8 warps poly (no clamp)", 16);
    run<2, true, false, 1, 0, 10>("TS+SS + 8 warps poly (clamp)", 16);
    run<2, true, false, 1, 0, 11>("TS+SS + 8 warps MUFU+FFMA2", 16);
    run<2, true, false, 1, 0, 12>("TS+SS + 8 warps FMNMX+FMUL", 16);
    run<2, true, false, 1, 0, 13>("TS+SS + 8 warps shl+add", 16);
    return 0;
  }
  run<0, false, false>("2CTA SS M256 N128 zeros", 8);
  run<0, true, false>("2CTA SS M256 N128 random", 8);
  run<1, true, false>("2CTA TS M256 N128 random", 8);
  run<2, false, false>("2CTA TS+SS zeros", 16);
  run<2, true, false>("2CTA TS+SS random", 16);
  run<2, true, true>("2CTA TS+SS random+TMEM ld/st", 16);
  run<0, true, false, 1>("2CTA SS + commit per 8 MMAs", 8);
  run<2, true, false, 1>("2CTA TS+SS + commit per 16", 16);
  run<2, true, false, 1, 1>("... + fence::after per 16", 16);
  run<2, true, false, 1, 2>("... + mbar try_wait per 16", 16);
  run<2, true, false, 1, 3>("... + both per 16", 16);
  run<2, true, false, 1, 0, 1>("TS+SS + 8 warps MUFU math", 16);
  run<2, true, false, 1, 0, 2>("TS+SS + 8 warps MUFU+poly math", 16);
  run<2, true, false, 1, 0, 3>("TS+SS + 8 warps FFMA", 16);
  run<2, true, false, 1, 0, 4>("TS+SS + 8 warps FFMA2", 16);
  run<2, true, false, 1, 0, 5>("TS+SS + 8 warps F2FP", 16);
  run<2, true, false, 1, 0, 6>("TS+SS + 8 warps MUFU.EX2", 16);
  run<2, true, false, 1, 0, 7>("TS+SS + 8 warps FADD2", 16);
  run<2, true, false, 1, 0, 8>("TS+SS + 8 warps IMAD", 16);
  run<2, true, false, 1, 0, 9>("TS+SS + 8 warps poly (no clamp)", 16);
  run<2, true, false, 1, 0, 10>("TS+SS + 8 warps poly (clamp)", 16);
  run<2, true, false, 1, 0, 11>("TS+SS + 8 warps MUFU+FFMA2", 16);
  run<2, true, false, 1, 0, 12>("TS+SS + 8 warps FMNMX+FMUL", 16);
  run<2, true, false, 1, 0, 13>("TS+SS + 8 warps shl+add", 16);
  run<1, true, false, 1, 0, 4>("TS only + 8 warps FFMA2", 8);
  run<0, true, false, 1, 0, 4>("SS only + 8 warps FFMA2", 8);
  return 0;
}
