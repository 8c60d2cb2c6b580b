// exp_bench.cu -- throughput of the K2 softmax exponential block in isolation: W warps per
// SM each run one variant over 128 scores per iteration (the per-warp work of one
// ping-pong step), no MMA, no TMEM.  Reports SM cycles per 128-element block per warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_15922_b200/csrc tools/exp_bench.cu -o tools/exp_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace dz;

// V: 0 = K2 code (kPoly of 8 pairs on the polynomial), 1 = no row sum, 2 = no bf16 pack,
//    3 = MUFU only (no sum, no pack), 4 = scalar FADD row sum instead of FADD2
template <int kPoly, int V>
__device__ __forceinline__ void exp_block(const float* s, uint32_t (&pk)[32], uint64_t (&acc)[4], float (&accs)[4]) {
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    uint64_t x = ptx::f2_pack(s[2 * i], s[2 * i + 1]);
    uint64_t p;
    float p0, p1;
    if ((i % 8) >= 8 - kPoly) {
      p = ptx::f2_exp2_poly<false>(x);
      ptx::f2_unpack(p, p0, p1);
    } else {
      float x0, x1;
      ptx::f2_unpack(x, x0, x1);
      p0 = ptx::ex2(x0);
      p1 = ptx::ex2(x1);
      p = ptx::f2_pack(p0, p1);
    }
    if (V == 0 || V == 2) acc[i % 4] = ptx::f2_add(acc[i % 4], p);
    if (V == 4) accs[i % 4] += p0 + p1;
    if (V == 0 || V == 1 || V == 4) pk[i] = ptx::pack_bf16x2(p0, p1);
    else pk[i] = __float_as_uint(p0) ^ __float_as_uint(p1);
  }
}

// V 5: two phases -- all exponentials of the 32 pairs first, then row sums and bf16 packs
template <int kPoly>
__device__ __forceinline__ void exp_block2(const float* s, uint32_t (&pk)[32], uint64_t (&acc)[4]) {
  uint64_t pp[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    uint64_t x = ptx::f2_pack(s[2 * i], s[2 * i + 1]);
    if ((i % 8) >= 8 - kPoly) {
      pp[i] = ptx::f2_exp2_poly<false>(x);
    } else {
      pp[i] = ptx::f2_pack(ptx::ex2(s[2 * i]), ptx::ex2(s[2 * i + 1]));
    }
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    acc[i % 4] = ptx::f2_add(acc[i % 4], pp[i]);
    float p0, p1;
    ptx::f2_unpack(pp[i], p0, p1);
    pk[i] = ptx::pack_bf16x2(p0, p1);
  }
}

template <int kPoly, int V>
__global__ void bench(int iters, long long* cyc, uint32_t* sink) {
  float s[128];
  for (int i = 0; i < 128; ++i) s[i] = ((threadIdx.x * 131 + i * 17) % 61) - 30.5f;
  uint32_t x = 0;
  float l = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint64_t acc[4] = {0, 0, 0, 0};
    float accs[4] = {0, 0, 0, 0};
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      uint32_t pk[32];
      if (V == 5)
        exp_block2<kPoly>(s + 64 * half, pk, acc);
      else
        exp_block<kPoly, V>(s + 64 * half, pk, acc, accs);
#pragma unroll
      for (int i = 0; i < 32; ++i) x ^= pk[i];
    }
    const uint64_t a = ptx::f2_add(ptx::f2_add(acc[0], acc[1]), ptx::f2_add(acc[2], acc[3]));
    float a0, a1;
    ptx::f2_unpack(a, a0, a1);
    l += a0 + a1 + accs[0] + accs[1] + accs[2] + accs[3];
    s[it & 127] += 1e-3f;  // keep the loop honest
  }
  long long t1 = clock64();
  if (threadIdx.x % 32 == 0) cyc[blockIdx.x * 32 + threadIdx.x / 32] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = x ^ __float_as_uint(l);
}

template <int kPoly, int V>
void run(const char* name) {
  long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 148 * 32 * sizeof(long long));
  cudaMalloc(&sink, 148 * 1024 * sizeof(uint32_t));
  const int iters = 1000;
  printf("%-34s", name);
  for (int w : {4, 8, 16}) {
    bench<kPoly, V><<<148, w * 32>>>(10, cyc, sink);
    bench<kPoly, V><<<148, w * 32>>>(iters, cyc, sink);
    cudaDeviceSynchronize();
    long long h[148 * 32];
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int b = 0; b < 148; ++b) avg += h[b * 32];
    avg /= 148;
    printf(" | %d/SMSP: %6.0f per warp, %5.0f per SMSP", w / 4, avg / iters, avg / iters / (w / 4));
  }
  printf("  (%s)\n", cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  run<2, 0>("K2 block (poly 2/8)");
  run<2, 5>("two-phase (poly 2/8)");
  run<4, 5>("two-phase (poly 4/8)");
  run<0, 5>("two-phase (all MUFU)");
  run<0, 0>("all MUFU");
  run<1, 0>("poly 1/8");
  run<3, 0>("poly 3/8");
  run<4, 0>("poly 4/8");
  run<2, 1>("poly 2/8, no row sum");
  run<2, 2>("poly 2/8, no bf16 pack");
  run<2, 3>("poly 2/8, exp only");
  run<2, 4>("poly 2/8, scalar row sum");
  run<0, 3>("MUFU exp only");
  return 0;
}
