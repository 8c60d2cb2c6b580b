// rmsrope.cuh -- the arithmetic of the fused per-head RMSNorm + 3D RoPE (BJ:5; DESIGN.md readings
// A1-A9), shared by the prologue kernels (K1 / K4, prologue.cu) and the attention kernel's
// in-kernel Q conversion (attention.cu), so Q' has the same bits whichever kernel computes it
// (the Ulysses path converts Q in K1, the one-GPU path in K2).
//
//   x'_i = RoPE( x_i / sqrt(mean_j x_j^2 + eps) * g_i ) * sc
//
// A row of D elements is handled as D/8 chunks of 8.  Chunk partial sums of squares are fma
// chains from 0; they are combined as a butterfly over the chunks of each half-row (D/16 chunks),
// then the two half-rows are added: for D = 128, half = ((p0+p4)+(p2+p6))+((p1+p5)+(p3+p7)).
// Products are rounded individually (no contraction), so both kernels produce identical bits.
#pragma once
#include <cuda_fp16.h>
#include <cstdint>

namespace dz {
namespace rr {

__device__ __forceinline__ void bf16x8_to_f32(const uint4& v, float (&f)[8]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}

// sum of squares of one 8-element chunk
__device__ __forceinline__ float chunk_ss(const float (&f)[8]) {
  float s = 0.f;
#pragma unroll
  for (int e = 0; e < 8; ++e) s = fmaf(f[e], f[e], s);
  return s;
}

// the half-row combination of N chunk partials (in place; result in p[0]), the same tree as the
// shuffle butterfly of the prologue over strides N/2, ..., 1
template <int N>
__device__ __forceinline__ float half_sum(float (&p)[N]) {
#pragma unroll
  for (int m = N / 2; m >= 1; m >>= 1)
#pragma unroll
    for (int k = 0; k < m; ++k) p[k] = __fadd_rn(p[k], p[k + m]);
  return p[0];
}

__device__ __forceinline__ float inv_rms(float ss, int D, float eps) {
  return rsqrtf(__fadd_rn(__fmul_rn(ss, 1.0f / (float)D), eps));
}

__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// one rotation pair (x_{2i}, x_{2i+1}) of an axis slice: normalised, times the gains, rotated by
// (cos, sin), times sc; fp16 pair
__device__ __forceinline__ uint32_t rot_pair(float f0, float f1, float inv, float g0, float g1, float2 cs, float sc) {
  const float u = __fmul_rn(__fmul_rn(f0, inv), g0);
  const float x = __fmul_rn(__fmul_rn(f1, inv), g1);
  const float a = __fmul_rn(__fsub_rn(__fmul_rn(u, cs.x), __fmul_rn(x, cs.y)), sc);
  const float b = __fmul_rn(__fadd_rn(__fmul_rn(u, cs.y), __fmul_rn(x, cs.x)), sc);
  return pack_half2(a, b);
}

// FP8 (E4M3) form of rot_pair: the rotated pair times sc, then times f8 (a power of two), rounded to
// nearest E4M3 with saturation; two bytes (lo = element 2i, hi = element 2i+1)
__device__ __forceinline__ uint16_t rot_pair_e4m3(float f0, float f1, float inv, float g0, float g1, float2 cs,
                                                  float sc, float f8) {
  const float u = __fmul_rn(__fmul_rn(f0, inv), g0);
  const float x = __fmul_rn(__fmul_rn(f1, inv), g1);
  const float a = __fmul_rn(__fmul_rn(__fsub_rn(__fmul_rn(u, cs.x), __fmul_rn(x, cs.y)), sc), f8);
  const float b = __fmul_rn(__fmul_rn(__fadd_rn(__fmul_rn(u, cs.y), __fmul_rn(x, cs.x)), sc), f8);
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(b), "f"(a));
  return r;
}

// (cos, sin) of the angle p * omega in fp64, rounded to fp32 (the RoPE table's values; used in place
// for positions beyond the table)
__device__ __noinline__ inline float2 rope_cs(int p, double omega) {
  double sn, cn;
  sincos((double)p * omega, &sn, &cn);
  return make_float2((float)cn, (float)sn);
}

}  // namespace rr
}  // namespace dz
