// pipe_bench.cu -- per-SM throughput of the softmax building blocks on sm_100a:
// FFMA, FFMA2, FADD2, MUFU.EX2, F2FP (cvt.rn.bf16x2.f32), IMAD-shift, FMNMX.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_15922_b200/csrc tools/pipe_bench.cu -o tools/pipe_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace dz;

template <int OP>
__global__ void __launch_bounds__(256) bench(float* out, int iters, long long* cyc) {
  float a[8];
  uint64_t v[8];
  uint32_t u[8];
  for (int i = 0; i < 8; ++i) {
    a[i] = threadIdx.x * 0.001f + i;
    v[i] = ptx::f2_pack(a[i], a[i] + 1.f);
    u[i] = threadIdx.x + i;
  }
  const uint64_t c2 = ptx::f2_pack(0.999f, 0.999f), d2 = ptx::f2_pack(0.001f, 0.001f);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) a[i] = fmaf(a[i], 0.999f, a[(i + 1) & 7]);
      if (OP == 1) v[i] = ptx::f2_fma(v[i], c2, d2);
      if (OP == 2) v[i] = ptx::f2_add(v[i], d2);
      if (OP == 3) a[i] = ptx::ex2(a[i]) - 0.5f;
      if (OP == 4) u[i] = ptx::pack_bf16x2(__uint_as_float(u[i]), a[i]);
      if (OP == 5) u[i] = __float_as_uint(a[i]) + (u[i] << 23);
      if (OP == 6) a[i] = fmaxf(fmaxf(a[i], a[(i + 1) & 7]), a[(i + 2) & 7]);
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) {
    float x, y;
    ptx::f2_unpack(v[i], x, y);
    s += a[i] + x + y + __uint_as_float(u[i]);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int warps_per_block) {
  float* o;
  long long* c;
  cudaMalloc(&o, 148 * 1024 * sizeof(float));
  cudaMalloc(&c, 148 * sizeof(long long));
  const int iters = 20000;
  bench<OP><<<148, warps_per_block * 32>>>(o, 100, c);
  bench<OP><<<148, warps_per_block * 32>>>(o, iters, c);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  // cycles per warp-instruction per SMSP: total cycles / (instructions issued per SMSP)
  const double instr_per_smsp = (double)iters * 8 * warps_per_block / 4;
  printf("%-22s warps/SMSP %d: %6.2f cycles per warp-instruction per SMSP  (%s)\n", name, warps_per_block / 4,
         avg / instr_per_smsp, cudaGetErrorString(cudaGetLastError()));
  cudaFree(o);
  cudaFree(c);
}

int main() {
  for (int w : {4, 8}) {
    run<0>("FFMA", w);
    run<1>("FFMA2", w);
    run<2>("FADD2", w);
    run<3>("MUFU.EX2 (+FADD)", w);
    run<4>("F2FP bf16x2", w);
    run<5>("shl+add (exp field)", w);
    run<6>("FMNMX3", w);
  }
  return 0;
}
