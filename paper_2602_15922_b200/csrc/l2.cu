// Benchmark helper (not on the hot path): drop a buffer's lines from L2 without writing them back.
//
// bench.py flushes L2 before every timed step by writing a 512 MB buffer.  The write leaves the
// last ~126 MB of that buffer in L2 as DIRTY lines, which the step's own loads must then evict --
// 126 MB of write-back traffic that belongs to the flush, not to the step.  `discard.global.L2`
// invalidates a 128-byte line without a write-back (the line's contents become undefined, which is
// fine for a scratch buffer), so write + discard leaves an L2 that holds none of the step's inputs
// and nothing to write back: the state a cold start (or ncu's cache control) gives.
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.h"

namespace dz {
namespace {

__global__ void l2_discard_kernel(char* __restrict__ p, size_t lines) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < lines; i += (size_t)gridDim.x * blockDim.x)
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p + i * 128) : "memory");
}

}  // namespace

cudaError_t launch_l2_discard(void* p, size_t bytes, cudaStream_t s) {
  const size_t lines = bytes / 128;
  if (lines == 0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  l2_discard_kernel<<<sms * 8, 256, 0, s>>>(static_cast<char*>(p), lines);
  return cudaGetLastError();
}

}  // namespace dz
