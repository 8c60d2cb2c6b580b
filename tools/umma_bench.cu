// umma_bench.cu -- microbenchmark of tcgen05.mma throughput on one SM (all SMs in parallel).
// Measures cycles per MMA instruction for SS (A,B smem) and TS (A tmem) kind::f16 shapes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2602_15922_b200/csrc tools/umma_bench.cu -o /tmp/umma_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace dz;

template <int MODE, int N>  // MODE 0: SS, 1: TS (A from TMEM), 2: SS two accumulators, 3: TS+SS interleaved,
                            // 4: mode 3 + 4 warps streaming tcgen05.ld/st (softmax-like TMEM traffic)
__global__ void __launch_bounds__(256, 1) bench(long long* cycles, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  // zero-fill 96 KB of operands
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem_raw + (base - raw))[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    ptx::mbar_init(ptx::smem_u32(&bar), 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc<512>(ptx::smem_u32(&tbase));
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc_ss = ptx::idesc_f16(0, 0, 0, 0, 128, N);
    constexpr uint32_t idesc_ts = ptx::idesc_f16(1, 1, 0, 1, 128, N);
    const uint32_t a = base, b = base + 32768;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk / 4) * 16384 + (kk % 4) * 32;
        if (MODE == 0)
          ptx::mma_ss(tmem, ptx::sdesc_sw128(a + off, 16, 1024), ptx::sdesc_sw128(b + off, 16, 1024), idesc_ss, 1);
        else if (MODE == 1)
          ptx::mma_ts(tmem + 256, tmem + kk * 8, ptx::sdesc_sw128(b + kk * 2048, 16384, 1024), idesc_ts, 1);
        else if (MODE == 2)
          ptx::mma_ss(tmem + (it & 1) * 256, ptx::sdesc_sw128(a + off, 16, 1024),
                      ptx::sdesc_sw128(b + off, 16, 1024), idesc_ss, 1);
      }
      if (MODE >= 3) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          ptx::mma_ts(tmem + 256, tmem + kk * 8, ptx::sdesc_sw128(b + kk * 2048, 16384, 1024), idesc_ts, 1);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk / 4) * 16384 + (kk % 4) * 32;
          ptx::mma_ss(tmem + 128, ptx::sdesc_sw128(a + off, 16, 1024), ptx::sdesc_sw128(b + off, 16, 1024),
                      idesc_ss, 1);
        }
      }
    }
    ptx::tc_commit(ptx::smem_u32(&bar));
    ptx::mbar_wait(ptx::smem_u32(&bar), 0);
    long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
    *(volatile int*)&tbase = -1;  // stop the TMEM streamers
  }
  if (MODE == 4 && warp >= 4) {
    const uint32_t lanes = (uint32_t)((warp % 4) * 32) << 16;
    uint32_t r[32];
    for (int k = 0; k < 200000 && *(volatile int*)&tbase != -1; ++k) {
      ptx::tmem_ld32(tmem + lanes + 384 + (k & 3) * 32, r);
      ptx::tmem_wait_ld();
      ptx::tmem_st32(tmem + lanes + 384 + ((k + 1) & 3) * 32, r);
      ptx::tmem_wait_st();
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 0) ptx::tmem_dealloc<512>(tmem);
}

template <int MODE, int N>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  const int iters = 4096;
  auto k = bench<MODE, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<<<148, 256, 100 * 1024>>>(d, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<148, 256, 100 * 1024>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double instrs = iters * (MODE >= 3 ? 16.0 : 8.0);
  const double flop = 148.0 * instrs * 2.0 * 128 * N * 16;
  printf("%-28s cyc/instr %7.2f  (ideal %5.1f)  %8.1f TFLOP/s  err=%s\n", name, avg / instrs, 128.0 * N / 256,
         flop / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<0, 128>("SS M128 N128 K16");
  run<0, 256>("SS M128 N256 K16");
  run<0, 64>("SS M128 N64 K16");
  run<1, 128>("TS M128 N128 K16");
  run<1, 256>("TS M128 N256 K16");
  run<2, 128>("SS M128 N128 alt acc");
  run<3, 128>("TS+SS N128 interleaved");
  run<4, 128>("TS+SS + TMEM ld/st traffic");
  return 0;
}
