// prologue.cu -- K1 (attend) / K4 (append): fused per-head RMSNorm + 3D RoPE.
//
//   x'_i = RoPE_3D( x_i / sqrt(mean_j x_j^2 + eps) * g_{h,i} )   for Q and K,
//   V copied unchanged,
// per (token, head) row of D elements (BJ:5 "per-head RMSNorm on Q/K and 3D
// (frame, height, width) RoPE"; readings A1-A9 in DESIGN.md: interleaved pairs
// (2i, 2i+1) inside the axis slices [t | h | w], omega_i = theta^(-2i/d_a)).
// fp32 math; Q' and K' stored fp16 (reading A13), V stays bf16.  Q' is stored
// multiplied by softmax_scale * log2(e), so the attention kernel's scores come
// out of the tensor core already in log2 units (one FMA per score saved).
//
// Layout: one CTA per (token, batch element).  Every thread first issues
// all of its 16-byte loads for the token (3 tensors x kPer heads in flight), and
// only then do two warps compute the token's D/2 rotation angles (fp64 sincos
// of p_a * omega_j) into shared memory, so the angle latency hides under the
// HBM latency instead of preceding it.  A row is handled by D/8 threads with
// one 16-byte load and one 16-byte store each; the row's sum of squares is
// reduced with __shfl_xor inside that thread group.  Heads are walked with
// loop counters (no runtime integer division per row).  HBM-bound by design: per
// token it moves (read + write) 2 B x D x H for each of Q, K, V.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.h"

namespace dz {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ void bf16x8_to_f32(const uint4& v, float (&f)[8]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}

// read-once activations: non-coherent path, no L1 allocation
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <int D>
__global__ void __launch_bounds__(kThreads) prologue_kernel(const PrologueArgs a) {
  constexpr int G = D / 8;             // threads per row (one 16-byte vector each)
  constexpr int kGroups = kThreads / G;  // rows processed side by side
  constexpr int kPer = 3;              // heads per thread and tensor in one pass
  __shared__ float2 cs[D / 2];         // (cos, sin) per pair of this token
  const int t = blockIdx.x;
  const int b = blockIdx.y;
  const int tid = threadIdx.x;
  const int g = tid / G;               // row group
  const int li = tid % G;              // 8-element slice index inside the row
  const int H = a.H;
  const int64_t xrow0 = (int64_t)b * a.x_bstride + (int64_t)t * H * D;

  // passes over blocks of kGroups * kPer heads (one pass for H <= 48 at D = 128); the trip
  // count is block-uniform, so the __syncthreads below is reached by every thread
  for (int h0 = 0; h0 < H; h0 += kGroups * kPer) {
    uint4 in[3][kPer];
#pragma unroll
    for (int w = 0; w < 3; ++w)
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const int h = h0 + g + k * kGroups;
        const uint4* src = reinterpret_cast<const uint4*>(a.x[w]);
        in[w][k] = (src != nullptr && h < H) ? ld_stream(src + (xrow0 + (int64_t)h * D) / 8 + li)
                                             : make_uint4(0, 0, 0, 0);
      }
    if (h0 == 0) {  // the token's rotation angles while the loads are in flight
      if (tid < D / 2) {
        const double p = (double)__ldg(a.pos + 3 * t + a.axis[tid]);
        double sn, cn;
        sincos(p * a.omega[tid], &sn, &cn);
        cs[tid] = make_float2((float)cn, (float)sn);
      }
      __syncthreads();
    }
    int64_t row_off[kPer];  // output row offset (without the tensor base) of head h
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int h = h0 + g + k * kGroups;
      const int dest = h / a.heads_per_dest, hl = h - dest * a.heads_per_dest;
      row_off[k] = (int64_t)dest * a.y[0].dstride + (int64_t)hl * D;  // dstride is the same for q, k, v slots
    }
#pragma unroll
    for (int w = 0; w < 3; ++w) {
      if (a.x[w] == nullptr) continue;  // block-uniform
      const OutSlot& o = a.y[w];
      const int64_t base = (int64_t)b * o.bstride + (int64_t)t * o.tstride;
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const int h = h0 + g + k * kGroups;
        if (w == 2) {  // V: unchanged bf16 copy into the cache / send slot
          if (h < H) reinterpret_cast<uint4*>(o.base)[(base + row_off[k]) / 8 + li] = in[w][k];
          continue;
        }
        float f[8];
        bf16x8_to_f32(in[w][k], f);
        float ss = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) ss = fmaf(f[i], f[i], ss);
        // every lane takes part (the two row groups of a warp may differ in validity)
#pragma unroll
        for (int m = G / 2; m >= 1; m >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, m);
        if (h >= H) continue;
        const float inv = rsqrtf(ss * (1.0f / D) + a.eps);
        const float4* gp = reinterpret_cast<const float4*>(a.gain[w] + h * D + li * 8);
        const float4 g0 = __ldg(gp), g1 = __ldg(gp + 1);
        const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
        const float sc = w == 0 ? a.q_scale : 1.f;  // Q' leaves pre-scaled by softmax_scale*log2(e)
        uint32_t pk[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float u = f[2 * i] * inv * gg[2 * i];
          const float v = f[2 * i + 1] * inv * gg[2 * i + 1];
          const float2 c = cs[li * 4 + i];
          pk[i] = pack_half2((u * c.x - v * c.y) * sc, (u * c.y + v * c.x) * sc);
        }
        reinterpret_cast<uint4*>(o.base)[(base + row_off[k]) / 8 + li] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      }
    }
  }
}

}  // namespace

cudaError_t launch_prologue(const PrologueArgs& a, cudaStream_t s) {
  if (a.n == 0 || a.B == 0) return cudaSuccess;
  dim3 grid(a.n, a.B);
  if (a.D == 128)
    prologue_kernel<128><<<grid, kThreads, 0, s>>>(a);
  else if (a.D == 64)
    prologue_kernel<64><<<grid, kThreads, 0, s>>>(a);
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

// K5: [N src][B][n_loc][Hl][D] -> [B][n_loc][H = N*Hl][D], one 16-byte vector per thread.
__global__ void sp_unpack_kernel(const uint4* __restrict__ recv, uint4* __restrict__ out, int N, int B, int n_loc,
                                 int Hl, int vec_per_row) {
  const int64_t total = (int64_t)N * B * n_loc * Hl * vec_per_row;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i;
    const int v = r % vec_per_row; r /= vec_per_row;
    const int hl = r % Hl; r /= Hl;
    const int t = r % n_loc; r /= n_loc;
    const int b = r % B; r /= B;
    const int src = (int)r;
    const int64_t o = (((int64_t)b * n_loc + t) * (N * Hl) + (int64_t)src * Hl + hl) * vec_per_row + v;
    out[o] = recv[i];
  }
}

cudaError_t launch_sp_unpack(const void* recv, void* out, int32_t N, int32_t B, int32_t n_loc, int32_t Hl, int32_t D,
                             cudaStream_t s) {
  const int vpr = D / 8;
  const int64_t total = (int64_t)N * B * n_loc * Hl * vpr;
  if (total == 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((total + threads - 1) / threads, 148 * 16);
  sp_unpack_kernel<<<(unsigned)blocks, threads, 0, s>>>(static_cast<const uint4*>(recv), static_cast<uint4*>(out), N,
                                                        B, n_loc, Hl, vpr);
  return cudaGetLastError();
}

}  // namespace dz
