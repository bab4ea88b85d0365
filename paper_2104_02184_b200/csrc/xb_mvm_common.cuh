// xb_mvm_common.cuh -- the MVM output stage shared by the stand-alone
// epilogue kernel (xb_mvm.cu) and the cluster-fused tcgen05 epilogue
// (xb_mvm_tc.cu), so both produce bit-identical outputs.
//
// v = acc + sigma_w ||x~|| zeta + sigma_out xi;  y = alpha 2^m Q_adc(v);
// zero-input samples get Q_adc(sigma_out xi) only (proj/src/io.cpp:107-115,
// 126-146).  Output noise: one Philox call per GROUP of 4 consecutive global
// outputs (counter = group, sample sequence number, BM exponent, tag); output
// 4g + k takes word k = two 16-bit Box-Muller normals (z0 -> sigma_w fold,
// z1 -> sigma_out).  Keyed on global indices: shards reproduce the tile.
#pragma once

#include "xb_internal.h"

namespace xb {

// per-sample state of one MVM call: alpha (0 = zero input), norm of x~,
// current BM exponent m, active flag for the current pass
struct SampleState {
  float alpha;
  float norm;
  int m;
  int active;
};

// 2^m exactly (0 <= m < 1023) from the exponent field, not the fp64 exp2 routine
__device__ __forceinline__ double pow2i(int m) {
  return __longlong_as_double((long long)(1023 + m) << 52);
}

__device__ __forceinline__ void out_noise_words(uint32_t g, uint64_t seq, int m, Key key,
                                                uint32_t w[4]) {
  uint32_t c0 = g, c1 = (uint32_t)seq, c2 = (uint32_t)(seq >> 32) | ((uint32_t)m << 24),
           c3 = TAG_OUT_NOISE << 24;
  philox10(c0, c1, c2, c3, key);
  w[0] = c0;
  w[1] = c1;
  w[2] = c2;
  w[3] = c3;
}

// groups of 4 global outputs covering [o0, o0 + M)
__host__ __device__ __forceinline__ int out_groups(int o0, int M) {
  return ((o0 + M - 1) >> 2) - (o0 >> 2) + 1;
}

// Outputs 4g..4g+3 (global index) of one sample: a[k] = their contraction
// sums; the ones inside [o0, o0 + M) are written to yrow[o - o0].  Returns
// whether any of them reached the ADC bound (bound management).
__device__ __forceinline__ bool epilogue_group4(const float a[4], int g, int o0, int M,
                                                const SampleState &s, const IoDev &io, Key key,
                                                uint64_t seq, float *__restrict__ yrow) {
  uint32_t w[4] = {0u, 0u, 0u, 0u};
  const bool noisy = !io.perfect && (io.sigma_w > 0.0 || io.sigma_out > 0.0);
  if (noisy) out_noise_words((uint32_t)g, seq, s.m, key, w);
  bool hit = false;
  if (!io.exact && !io.perfect) {
    // fp32 output stage (tensor-core modes): alpha 2^m y rounds once in fp32,
    // exactly like the fp64 product cast to fp32 (2^m is exact)
    const float scale = s.alpha == 0.f ? 1.f : s.alpha * (float)pow2i(s.m);
    const float sw = (float)io.sigma_w * s.norm, so = (float)io.sigma_out;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int o = 4 * g + k - o0;
      if (o < 0 || o >= M) continue;
      float z0 = 0.f, z1 = 0.f;
      if (noisy) box_muller16(w[k], z0, z1);
      float v;
      if (s.alpha == 0.f) {
        v = so * z1;
      } else {
        v = a[k];
        if (io.sigma_w > 0.0) v = fmaf(sw, z0, v);
        v = fmaf(so, z1, v);
        hit |= fabsf(v) >= io.adc.fbound;
      }
      yrow[o] = scale * quantize_f(v, io.adc);
    }
    return hit;
  }
  const double scale = s.alpha == 0.f ? 1.0 : (double)s.alpha * pow2i(s.m);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int o = 4 * g + k - o0;
    if (o < 0 || o >= M) continue;
    if (io.perfect) {
      yrow[o] = a[k];
      continue;
    }
    float z0 = 0.f, z1 = 0.f;
    if (noisy) box_muller16(w[k], z0, z1);
    double v;
    if (s.alpha == 0.f) {
      v = io.sigma_out > 0.0 ? io.sigma_out * (double)z1 : 0.0;
    } else {
      v = (double)a[k];
      if (io.sigma_w > 0.0) v += io.sigma_w * (double)s.norm * (double)z0;
      if (io.sigma_out > 0.0) v += io.sigma_out * (double)z1;
      hit |= fabs(v) >= io.adc.bound;
    }
    yrow[o] = (float)(scale * quantize(v, io.adc));
  }
  return hit;
}

// BM bookkeeping: one flag write per warp (a saturating sample saturates many
// outputs; per-thread atomics on the same word would serialise)
__device__ __forceinline__ void bm_flag(bool hit, const SampleState &s, const IoDev &io,
                                        int *sat, int b, int B, int pass_slot) {
  if (io.bm && s.alpha != 0.f && s.m < io.bm_max_iter) {
    const unsigned any = __ballot_sync(__activemask(), hit);
    if (hit && (threadIdx.x & 31) == __ffs(any) - 1 && atomicExch(sat + b, 1) == 0)
      atomicAdd(sat + B + pass_slot, 1);
  }
}

// arguments of the fused output stage
struct FusedOut {
  float *Y;            // [B][ldy]
  int ldy;
  const SampleState *st;
  IoDev io;
  Key key;
  uint64_t seq0;       // sequence number of sample 0 of the call
  int *sat;            // BM flags [B] + per-pass counters
  int first_pass, B, pass_slot;
  int o0;              // global index of output 0 (row shards: row0; backward: 0)
  int n0;              // first x~ row of this N slab
  const int *map;      // x~ row -> sample (compacted BM re-issue), or nullptr
};

// tcgen05 contraction (xb_mvm_tc.cu).  fo == nullptr: split-K partial sums
// part[s][b][o] (split stride B x M); otherwise the cluster-fused output stage
// writes fo->Y (requires fo->o0 % 4 == 0 and splits <= 8).
void tc_gemm(Tile &t, bool transposed, bool x3, const float *Xt, int ldt, int B, float *part,
             int splits, const FusedOut *fo);

} // namespace xb
