// l2bw_bench.cu -- L2 -> shared memory fill rate per SM with TMA bulk copies (1 CTA per SM,
// W issuing warps, each keeping DEPTH copies of BYTES in flight) from an L2-resident buffer.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_15922_b200/csrc tools/l2bw_bench.cu -o tools/l2bw_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace dz;

__global__ void __launch_bounds__(256, 1) fill(const uint8_t* src, size_t src_bytes, int W, int depth, int bytes,
                                               int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[8][8];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int w = 0; w < 8; ++w)
      for (int i = 0; i < 8; ++i) ptx::mbar_init(ptx::smem_u32(&bar[w][i]), 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const uint64_t pol = ptx::l2_policy_evict_last();
  long long t0 = clock64();
  if (warp < W && lane == 0) {
    uint32_t ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const uint32_t dst0 = ptx::smem_u32(sm) + warp * depth * bytes;
    size_t off = ((size_t)blockIdx.x * 7919 + warp * 104729) * 4096 % src_bytes;
    for (int k = 0; k < iters; ++k) {
      const int sl = k % depth;
      if (k >= depth) {
        ptx::mbar_wait(ptx::smem_u32(&bar[warp][sl]), ph[sl]);
        ph[sl] ^= 1;
      }
      ptx::mbar_arrive_expect_tx(ptx::smem_u32(&bar[warp][sl]), bytes);
      ptx::bulk_load(dst0 + sl * bytes, src + off, bytes, ptx::smem_u32(&bar[warp][sl]), pol);
      off += bytes;
      if (off + bytes > src_bytes) off = 0;
    }
    for (int k = iters; k < iters + depth; ++k) {
      const int sl = k % depth;
      ptx::mbar_wait(ptx::smem_u32(&bar[warp][sl]), ph[sl]);
      ph[sl] ^= 1;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  const size_t src_bytes = 32u << 20;  // 32 MB: L2-resident
  uint8_t* src;
  cudaMalloc(&src, src_bytes);
  cudaMemset(src, 1, src_bytes);
  long long* out;
  cudaMalloc(&out, 1024 * sizeof(long long));
  cudaFuncSetAttribute(fill, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int sms = 148;
  struct Cfg { int W, depth, bytes, grid; };
  const Cfg cfgs[] = {{1, 2, 16384, 148}, {1, 4, 16384, 148}, {2, 4, 16384, 148}, {4, 2, 16384, 148},
                      {4, 4, 8192, 148}, {8, 2, 8192, 148}, {2, 4, 16384, 74}, {2, 4, 16384, 16}, {2, 4, 16384, 1}};
  for (const Cfg& c : cfgs) {
    const int iters = 2000;
    fill<<<c.grid, 256, 200 * 1024>>>(src, src_bytes, c.W, c.depth, c.bytes, 50, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    fill<<<c.grid, 256, 200 * 1024>>>(src, src_bytes, c.W, c.depth, c.bytes, iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[1024];
    cudaMemcpy(h, out, sizeof(long long) * c.grid, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int b = 0; b < c.grid; ++b) avg += h[b];
    avg /= c.grid;
    const double per_cta = (double)c.W * (iters + c.depth) * c.bytes;
    printf("grid %3d W %d depth %d bytes %6d: %6.1f B/clk per SM, aggregate %7.1f GB/s (%s)\n", c.grid, c.W, c.depth,
           c.bytes, per_cta / avg, per_cta * c.grid / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  (void)sms;
  return 0;
}
