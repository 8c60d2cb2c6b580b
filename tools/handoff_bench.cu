// handoff_bench.cu -- latency of the MMA <-> softmax handshake on a CTA pair (no softmax math).
// Per step: MMA thread issues 8 SS MMAs (QK-like) for tile t, commits s_full[t] (multicast);
// 4 "softmax" warps per CTA per tile wait s_full[t], optionally tcgen05.ld 128 columns, arrive
// s_free (remote, leader) and p_full[t]; MMA thread waits p_full[t] (PV-like 8 TS MMAs) and s_free.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_15922_b200/csrc tools/handoff_bench.cu -o tools/handoff_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace dz;

struct B {
  uint64_t s_full[2], s_free, p_full[2], p_empty[2];
  uint32_t tmem;
};

template <int MODE>  // 0: QK only + handshake; 1: QK + PV interleaved + handshake; 2: mode 1 with local (non-2CTA)...
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1) bench(long long* cyc, int steps, int load_s) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  __shared__ B bb;
  B* bars = &bb;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = ptx::cluster_ctarank();
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem_raw + (base - raw))[i] = make_uint4(0x3c003c00u, 0x3c003c00u, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  auto bar = [&](uint64_t& b) { return ptx::smem_u32(&b); };
  auto lbar = [&](uint64_t& b) { return ptx::mapa(ptx::smem_u32(&b), 0); };
  if (threadIdx.x == 0) {
    ptx::mbar_init(bar(bars->s_free), 8);
    for (int t = 0; t < 2; ++t) {
      ptx::mbar_init(bar(bars->s_full[t]), 1);
      ptx::mbar_init(bar(bars->p_full[t]), 8);
      ptx::mbar_init(bar(bars->p_empty[t]), 1);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 8) ptx::tmem_alloc_2cta<512>(ptx::smem_u32(&bars->tmem));
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = bars->tmem;
  constexpr uint32_t idesc_ss = ptx::idesc_f16(0, 0, 0, 0, 256, 128);
  constexpr uint32_t idesc_ts = ptx::idesc_f16(1, 1, 0, 1, 256, 128);
  if (warp == 11 && rank == 0) {
    uint32_t sf = 0, pp[2] = {0, 0};
    long long t0 = clock64();
    for (int g = 0; g <= steps; ++g) {
      for (int t = 0; t < 2; ++t) {
        if (g < steps) {
          if (g > 0 || t > 0) {
            ptx::mbar_wait(bar(bars->s_free), sf);
            sf ^= 1;
          }
          ptx::tc_fence_after();
          if (lane == 0) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              ptx::mma_ss_2cta(tmem, ptx::sdesc_sw128(base + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024),
                               ptx::sdesc_sw128(base + 32768 + (kk / 4) * 8192 + (kk % 4) * 32, 16, 1024), idesc_ss,
                               kk > 0);
            ptx::tc_commit_2cta(bar(bars->s_full[t]), 3);
          }
          __syncwarp();
        }
        if (MODE >= 1 && g > 0) {
          ptx::mbar_wait(bar(bars->p_full[t]), pp[t]);
          pp[t] ^= 1;
          ptx::tc_fence_after();
          if (lane == 0) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              ptx::mma_ts_2cta(tmem + 256 + t * 128, tmem + 128 + t * 64 + kk * 8,
                               ptx::sdesc_sw128(base + 65536 + kk * 2048, 16, 1024), idesc_ts, 1);
            ptx::tc_commit_2cta(bar(bars->p_empty[t]), 3);
          }
          __syncwarp();
        }
      }
    }
    long long t1 = clock64();
    if (lane == 0) cyc[blockIdx.x / 2] = t1 - t0;
  } else if (warp < 8) {
    const int t = warp / 4;
    const uint32_t lanes = (uint32_t)((warp % 4) * 32) << 16;
    uint32_t sp = 0, pe = 0;
    for (int g = 0; g < steps; ++g) {
      ptx::mbar_wait(bar(bars->s_full[t]), sp);
      sp ^= 1;
      ptx::tc_fence_after();
      if (load_s) {
        uint32_t r[32];
        for (int c = 0; c < 4; ++c) ptx::tmem_ld32(tmem + lanes + c * 32, r);
        ptx::tmem_wait_ld();
        if (r[0] == 12345) cyc[200] = r[1];
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_cluster(lbar(bars->s_free));
      if (MODE >= 1) {
        ptx::mbar_wait(bar(bars->p_empty[t]), pe ^ 1);
        pe ^= 1;
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(lbar(bars->p_full[t]));
      }
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  if (warp == 8) ptx::tmem_dealloc_2cta<512>(tmem);
}

template <int MODE>
void run(const char* name, int load_s) {
  long long* d;
  cudaMalloc(&d, 256 * sizeof(long long));
  const int steps = 2000;
  auto k = bench<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<<<148, 384, 100 * 1024>>>(d, 20, load_s);
  k<<<148, 384, 100 * 1024>>>(d, steps, load_s);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[74];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 74; ++i) avg += h[i];
  avg /= 74;
  printf("%-40s load_s=%d: %8.1f cycles per step (2 tiles; ideal %d)  %s\n", name, load_s, avg / steps,
         MODE ? 2048 : 1024, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0>("QK only, S handshake", 0);
  run<0>("QK only, S handshake", 1);
  run<1>("QK+PV, S and P handshakes", 0);
  run<1>("QK+PV, S and P handshakes", 1);
  return 0;
}
