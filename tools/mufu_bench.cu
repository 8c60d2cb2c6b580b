// mufu_bench.cu -- exp2 throughput per SM for ex2.approx.ftz.f32 against the packed
// ex2.approx.f16x2 / ex2.approx.ftz.bf16x2 forms (two results per instruction): W warps per SM,
// each runs 8 independent chains of N exponentials.  Reports exponential RESULTS per clock per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mufu_bench.cu -o tools/mufu_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

template <int V>
__global__ void bench(float* out, long long* clk, float seed) {
  uint32_t r[8];
  float f[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    f[k] = -0.001f * (threadIdx.x + k) + seed;
    r[k] = 0x3c003c00u ^ (threadIdx.x + k);  // small positive halves
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (V == 0) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[k]));
      } else if (V == 1) {
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(r[k]));
      } else {
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(r[k]));
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) acc += f[k] + __uint_as_float(r[k]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int V>
void run(const char* name, int warps) {
  float* out;
  long long* clk;
  cudaMalloc(&out, 148 * 1024 * sizeof(float));
  cudaMalloc(&clk, 148 * sizeof(long long));
  bench<V><<<148, warps * 32>>>(out, clk, 0.5f);
  bench<V><<<148, warps * 32>>>(out, clk, 0.5f);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (long long x : h) mx = x > mx ? x : mx;
  const double results = (double)warps * 32 * kIters * 8 * (V == 0 ? 1 : 2);
  printf("%-22s warps/SM %2d: %.2f results/clk/SM (%.2f instr/clk/SM)\n", name, warps, results / mx,
         results / mx / (V == 0 ? 1 : 2));
  cudaFree(out);
  cudaFree(clk);
}

int main() {
  for (int w : {4, 8, 16, 32}) {
    run<0>("ex2.approx.ftz.f32", w);
    run<1>("ex2.approx.f16x2", w);
    run<2>("ex2.approx.ftz.bf16x2", w);
  }
  return 0;
}
