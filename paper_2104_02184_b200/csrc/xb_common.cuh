// xb_common.cuh -- shared device helpers for the B200 analog-tile kernels.
//
// Random numbers: counter-based Philox4x32-10 (Salmon et al., SC'11).  A
// stream is a 64-bit key derived from the tile seed with the reference's
// named-stream rule (RngStream::derive, proj/src/rng.cpp:35-41), and each
// draw is addressed by a 128-bit counter built from GLOBAL indices (sample
// sequence number, row, column, slot group).  Draws are therefore independent
// of launch geometry, batching into kernels and row sharding.
#pragma once

#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>

namespace xb {

struct Key {
  uint32_t k0, k1;
};

// ---------------------------------------------------------------- Philox
__host__ __device__ __forceinline__ void philox_round(uint32_t &c0, uint32_t &c1, uint32_t &c2,
                                                      uint32_t &c3, uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
#ifdef __CUDA_ARCH__
  const uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
  const uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
#else
  const uint64_t p0 = (uint64_t)M0 * c0, p1 = (uint64_t)M1 * c2;
  const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
  const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
  const uint32_t n0 = hi1 ^ c1 ^ k0;
  const uint32_t n2 = hi0 ^ c3 ^ k1;
  c0 = n0;
  c1 = lo1;
  c2 = n2;
  c3 = lo0;
}

// Philox4x32-10: counter (c0..c3), key (k0,k1) -> 4 x u32, in place.
__host__ __device__ __forceinline__ void philox10(uint32_t &c0, uint32_t &c1, uint32_t &c2,
                                                  uint32_t &c3, Key key) {
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  uint32_t k0 = key.k0, k1 = key.k1;
#pragma unroll
  for (int r = 0; r < 9; ++r) {
    philox_round(c0, c1, c2, c3, k0, k1);
    k0 += W0;
    k1 += W1;
  }
  philox_round(c0, c1, c2, c3, k0, k1);
}

// u32 -> float uniform in (0, 1]; never 0 so log() is finite
__device__ __forceinline__ float u01_open0(uint32_t u) {
  return fmaf((float)u, 2.3283064365386963e-10f, 1.1641532182693481e-10f);
}
// u32 -> float uniform in [0, 1)
__device__ __forceinline__ float u01(uint32_t u) { return (float)(u >> 8) * 5.9604644775390625e-8f; }

// Box-Muller: two u32 -> two N(0,1)
__device__ __forceinline__ void box_muller(uint32_t a, uint32_t b, float &z0, float &z1) {
  const float r = sqrtf(-2.0f * __logf(u01_open0(a)));
  float s, c;
  __sincosf(6.283185307179586f * u01(b), &s, &c);
  z0 = r * c;
  z1 = r * s;
}

// four standard normals from one Philox call
__device__ __forceinline__ void normal4(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                        Key key, float &z0, float &z1, float &z2, float &z3) {
  philox10(c0, c1, c2, c3, key);
  box_muller(c0, c1, z0, z1);
  box_muller(c2, c3, z2, z3);
}

// two standard normals from one Philox call (one Box-Muller pair)
__device__ __forceinline__ void normal2(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                        Key key, float &z0, float &z1) {
  philox10(c0, c1, c2, c3, key);
  box_muller(c0, c1, z0, z1);
}

__device__ __forceinline__ float normal1(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                         Key key) {
  philox10(c0, c1, c2, c3, key);
  float z0, z1;
  box_muller(c0, c1, z0, z1);
  return z0;
}

// two normals from one u32 (16-bit uniforms, half-LSB centred; MUFU
// approximations): the radius reaches sqrt(2 ln 2^17) = 4.9 sigma, a tail
// mass of 1e-6 that the noise statistics of this simulator cannot resolve
__device__ __forceinline__ void box_muller16(uint32_t a, float &z0, float &z1) {
  const float u = fmaf((float)(a & 0xffffu), 1.52587890625e-05f, 7.62939453125e-06f);
  const float th = fmaf((float)(a >> 16), 9.587379924285257e-05f, -3.1415446284412245f);
  float l, r, s, c;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(u));
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(l * -1.3862943611198906f)); // -2 ln u
  asm("sin.approx.ftz.f32 %0, %1;" : "=f"(s) : "f"(th));
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(c) : "f"(th));
  z0 = r * c;
  z1 = r * s;
}

// ------------------------------------------------------------ quantizer
// proj/src/io.cpp:42-56, evaluated in fp64 exactly as the reference does
// (the converters touch B x N values per call, never the MxN weight array):
// exact zero passes through, clamp, mid-rise grid -b + (k + 1/2) step with
// k = round-half-away((v + b - step/2) / step) clamped to [0, levels - 1].
struct Quant {
  double bound, step, inv_step, levels_m1;
  int bits;
  // fp32 copies for the tensor-core output stage (quantize_f)
  float fbound, fstep, finv_step, flevels_m1;
  int pow2; // bound is a power of two: every grid point is exact in fp32
};

__host__ __device__ __forceinline__ Quant make_quant(double bound, int bits) {
  Quant q;
  q.bound = bound;
  q.bits = bits;
  if (bits > 0) {
    const double levels = exp2((double)bits);
    q.step = 2.0 * bound / levels;
    q.inv_step = levels / (2.0 * bound);
    q.levels_m1 = levels - 1.0;
  } else {
    q.step = 0.0;
    q.inv_step = 0.0;
    q.levels_m1 = 0.0;
  }
  q.fbound = (float)q.bound;
  q.fstep = (float)q.step;
  q.finv_step = (float)q.inv_step;
  q.flevels_m1 = (float)q.levels_m1;
  int e = 0;
  q.pow2 = bound > 0.0 && bound < 1e30 && frexp(bound, &e) == 0.5;
  return q;
}

__device__ __forceinline__ double quantize(double v, const Quant &q) {
  if (v == 0.0) return 0.0;
  v = fmin(fmax(v, -q.bound), q.bound);
  if (q.bits <= 0) return v;
  // the reference divides by step; multiplying by its reciprocal differs by at
  // most one fp64 ulp, i.e. only on exact half-way ties of the grid
  double k = round((v + q.bound - 0.5 * q.step) * q.inv_step);
  k = fmin(fmax(k, 0.0), q.levels_m1);
  return -q.bound + (k + 0.5) * q.step;
}

// The same quantizer in fp32, for the output stage of the tensor-core MVM
// (TF32 / 3xTF32): its accumulators are fp32 already, so fp64 converter
// arithmetic there buys nothing but FP64-pipe time (the B200 runs fp64 at
// half the fp32 rate; the fused epilogue was bound by it).  The grid step is
// a power of two, so -b + (k + 1/2) step is exact in fp32; only inputs within
// ~1 fp32 ulp of a grid threshold can land one level away from the fp64
// quantizer, far below the TF32 contraction error.
__device__ __forceinline__ float quantize_f(float v, const Quant &q) {
  if (v == 0.f) return 0.f;
  v = fminf(fmaxf(v, -q.fbound), q.fbound);
  if (q.bits <= 0) return v;
  float k = roundf((v + q.fbound - 0.5f * q.fstep) * q.finv_step);
  k = fminf(fmaxf(k, 0.f), q.flevels_m1);
  return fmaf(k + 0.5f, q.fstep, -q.fbound);
}

// ------------------------------------------------------------ reductions
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Counter tags: the 4th counter word carries (tag << 24) | high bits of the
// sequence number so different draw families of one stream never collide.
enum : uint32_t {
  TAG_TRAIN_X = 1,
  TAG_TRAIN_D = 2,
  TAG_C2C = 3,
  TAG_IN_NOISE = 4,
  TAG_W_NOISE = 5,
  TAG_OUT_NOISE = 6,
  TAG_REALIZE = 7,
  TAG_PROGRAM = 8,
  TAG_NU = 9,
  TAG_TEMPORAL = 10,
  TAG_TEMPORAL_XI = 11,
};

__host__ __device__ __forceinline__ uint32_t tag_word(uint32_t tag, uint64_t seq) {
  return (tag << 24) | (uint32_t)((seq >> 32) & 0xFFFFFFu);
}

} // namespace xb
