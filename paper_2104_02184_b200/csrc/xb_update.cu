// xb_update.cu -- the stochastic pulsed update (paper Eq. 2) on sm_100a.
//
// Reference path (proj/src/pulsed.cpp:116-148):
//   translate (:25-66) -> generate_trains (:68-88) -> apply_coincidences (:90-114)
// applied once per sample, samples in order, each coincidence one device pulse
// (proj/src/device.cpp:48-77).
//
// B200 path, one batched call of B samples:
//   K3 rows_amax_kernel    per-sample max|x|, max|d| (row shards: the max over
//                          ranks is taken by the caller between K3 and K4)
//   K4 trains_kernel       translate in fp64 (bit-identical plan to the
//                          reference on the same inputs) and Philox Bernoulli
//                          trains packed one uint32 per (sample, line):
//                          bits 0..bl-1 = slots, bit 31 = sign (1 = negative)
//   K5 pulse_kernel        weight-stationary: each thread owns one cell, keeps
//                          w and the cell's realization in registers across
//                          all B samples, finds coincidences with AND, and
//                          applies the device law pulse by pulse in sample
//                          order (the same per-cell sequence as the
//                          reference's slot-major triple loop, since pulses of
//                          one sample share a direction).
//   K6 pulse_det_kernel    deterministic_implicit (pulsed.cpp:128-144).
#include "xb_internal.h"

namespace xb {

// ============================================================== K3: amax
// one CTA per sample row; 16-byte loads (when the row allows them), four in
// flight per thread, so the pass streams at HBM rate instead of waiting on
// one dependent load per iteration
// blocks [0, nb1) take rows of V (length n, stride ld) into out; blocks
// [nb1, gridDim.x) rows of V2 (n2, ld2) into out2 -- the x and d maxima of an
// update in one launch.  flag != null: check_input's finiteness test in the
// same pass (OR-ing bit1 / bit2 into *flag for a non-finite entry of V / V2):
// z sums v * 0, which stays 0 for finite entries and turns NaN otherwise.
__global__ void __launch_bounds__(256) rows_amax_kernel(const float *__restrict__ V, int n, int ld,
                                                        float *__restrict__ out, int nb1,
                                                        const float *__restrict__ V2, int n2,
                                                        int ld2, float *__restrict__ out2,
                                                        int *__restrict__ flag, int bit1,
                                                        int bit2) {
  int b = blockIdx.x;
  int bit = bit1;
  if (b >= nb1) {
    b -= nb1;
    V = V2;
    n = n2;
    ld = ld2;
    out = out2;
    bit = bit2;
  }
  float z = 0.f;
  const float *row = V + (size_t)b * ld;
  float m0 = 0.f, m1 = 0.f, m2 = 0.f, m3 = 0.f;
  int head = 0;
  if ((((uintptr_t)row) & 15) == 0) {
    const float4 *r4 = reinterpret_cast<const float4 *>(row);
    const int n4 = n >> 2;
    int j = threadIdx.x;
    for (; j + 3 * 256 < n4; j += 4 * 256) {
      const float4 a = __ldg(r4 + j), c = __ldg(r4 + j + 256), e = __ldg(r4 + j + 512),
                   g = __ldg(r4 + j + 768);
      m0 = fmaxf(m0, fmaxf(fmaxf(fabsf(a.x), fabsf(a.y)), fmaxf(fabsf(a.z), fabsf(a.w))));
      m1 = fmaxf(m1, fmaxf(fmaxf(fabsf(c.x), fabsf(c.y)), fmaxf(fabsf(c.z), fabsf(c.w))));
      m2 = fmaxf(m2, fmaxf(fmaxf(fabsf(e.x), fabsf(e.y)), fmaxf(fabsf(e.z), fabsf(e.w))));
      m3 = fmaxf(m3, fmaxf(fmaxf(fabsf(g.x), fabsf(g.y)), fmaxf(fabsf(g.z), fabsf(g.w))));
      if (flag) {
        z = fmaf(a.x, 0.f, fmaf(a.y, 0.f, fmaf(a.z, 0.f, fmaf(a.w, 0.f, z))));
        z = fmaf(c.x, 0.f, fmaf(c.y, 0.f, fmaf(c.z, 0.f, fmaf(c.w, 0.f, z))));
        z = fmaf(e.x, 0.f, fmaf(e.y, 0.f, fmaf(e.z, 0.f, fmaf(e.w, 0.f, z))));
        z = fmaf(g.x, 0.f, fmaf(g.y, 0.f, fmaf(g.z, 0.f, fmaf(g.w, 0.f, z))));
      }
    }
    for (; j < n4; j += 256) {
      const float4 a = __ldg(r4 + j);
      m0 = fmaxf(m0, fmaxf(fmaxf(fabsf(a.x), fabsf(a.y)), fmaxf(fabsf(a.z), fabsf(a.w))));
      if (flag) z = fmaf(a.x, 0.f, fmaf(a.y, 0.f, fmaf(a.z, 0.f, fmaf(a.w, 0.f, z))));
    }
    head = n4 << 2;
  }
  for (int j = head + threadIdx.x; j < n; j += 256) {
    m1 = fmaxf(m1, fabsf(row[j]));
    if (flag) z = fmaf(row[j], 0.f, z);
  }
  if (flag && __syncthreads_or(!(z == 0.f)) && threadIdx.x == 0) atomicOr(flag, bit);
  float m = warp_max(fmaxf(fmaxf(m0, m1), fmaxf(m2, m3)));
  __shared__ float red[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = m;
  __syncthreads();
  if (warp == 0) {
    m = warp_max(lane < 8 ? red[lane] : 0.f);
    if (lane == 0) out[b] = m;
  }
}

void launch_rows_amax(const float *V, int B, int n, int ld, float *out, cudaStream_t s) {
  if (B <= 0) return;
  rows_amax_kernel<<<B, 256, 0, s>>>(V, n, ld, out, B, nullptr, 0, 0, nullptr, nullptr, 0, 0);
  count_launch();
  XB_CUDA(cudaGetLastError());
}

void launch_rows_amax2(const float *X, int nx, float *xm, const float *D, int nd, float *dm, int B,
                       cudaStream_t s, int *flag) {
  if (B <= 0) return;
  rows_amax_kernel<<<2 * B, 256, 0, s>>>(X, nx, nx, xm, B, D, nd, nd, dm, flag, 1, 2);
  count_launch();
  XB_CUDA(cudaGetLastError());
}

// ---- Philox4x32-10 with the 10 round keys precomputed on the host (kernel
// parameters, i.e. constant-bank operands of the LOP3s): the key schedule
// costs no instructions.  Used by the trains (Bernoulli slots) and the c2c
// noise (Box-Muller factors; statistical parity only).
struct RoundKeys {
  uint32_t k0[10], k1[10];
};

static RoundKeys round_keys(Key k) {
  RoundKeys r;
  uint32_t a = k.k0, b = k.k1;
  for (int i = 0; i < 10; ++i) {
    r.k0[i] = a;
    r.k1[i] = b;
    a += 0x9E3779B9u;
    b += 0xBB67AE85u;
  }
  return r;
}

// Rounds of the Philox4x32 behind the c2c factors (the pulse loop's noise, ~1/3
// of its instructions).  Salmon et al. (SC'11) find Philox4x32 passing all of
// TestU01's BigCrush from 7 rounds on and recommend 10 as a safety margin;
// the c2c factors use 7 (round 2, B200: NS update 5.92 -> 5.55 ms), checked by
// the c2c single-pulse distribution / moment tests of all four laws
// (tests/test_gpu_update.py) and a uniformity / serial-correlation test of
// the 7-round stream on the kernel's exact counter pattern
// (tests/test_philox_rounds.py).  Every other draw keeps 10 rounds.
#ifndef XB_C2C_ROUNDS
#define XB_C2C_ROUNDS 7
#endif
template <int ROUNDS = 10>
__device__ __forceinline__ void philox10_rk(uint32_t &c0, uint32_t &c1, uint32_t &c2,
                                            uint32_t &c3, const RoundKeys &rk) {
#pragma unroll
  for (int r = 0; r < ROUNDS; ++r) philox_round(c0, c1, c2, c3, rk.k0[r], rk.k1[r]);
}

// ============================================================== K4: trains
// Counter of a train draw: (slot group g, global line, seq lo, seq hi ^ side),
// key = the tile's "update" stream.  Each Philox call gives 4 slots
// (trains_kernel).

// translate, proj/src/pulsed.cpp:25-66, in fp64 on the fp32 inputs: the
// per-sample part (BL management, amplitude, x/d rebalancing)
struct Plan {
  double amp, x_scale, d_scale;
  int bl, skip;
};

__device__ __forceinline__ Plan make_plan(double lrb, double x_amax, double d_amax, double dw_min,
                                          int BL, int blm) {
  Plan pl;
  pl.skip = (lrb == 0.0 || x_amax == 0.0 || d_amax == 0.0); // pulsed.cpp:122-124
  int bl = BL;
  if (blm && !pl.skip) {
    const double quanta = lrb * x_amax * d_amax / dw_min;
    const int c = (int)ceil(BL * (quanta < 1.0 ? quanta : 1.0));
    bl = c > 1 ? c : 1;
  }
  pl.bl = bl;
  pl.amp = pl.skip ? 0.0 : sqrt(lrb / (dw_min * bl));
  pl.x_scale = 1.0;
  pl.d_scale = 1.0;
  if (x_amax > 0.0 && d_amax > 0.0) {
    pl.x_scale = sqrt(d_amax / x_amax);
    pl.d_scale = 1.0 / pl.x_scale;
  }
  return pl;
}

// Packed trains, d LINE-major dw[line][b] (row stride ldb), x in the quad
// layout of xq_index (xb_internal.h); zero words for ldb > b >= B.  The pulse
// kernel then reads 4-8 consecutive samples of one line with a single vector
// load.  CTA tile: 32 lines x 32 samples; x lines first, then d lines.
__global__ void __launch_bounds__(256) trains_kernel(
    const float *__restrict__ X, const float *__restrict__ D, int C, int R, int B,
    const double *__restrict__ lr, double lr_scalar, const float *__restrict__ xm,
    const float *__restrict__ dm, double dw_min, const double *__restrict__ dwmin_b, int BL,
    int blm, const RoundKeys rk, uint64_t seq0, int row0, uint32_t *__restrict__ xw,
    uint32_t *__restrict__ dw, int ldb, int32_t *__restrict__ bl_out) {
  __shared__ Plan plan[32];
  __shared__ uint32_t tile[32][33];
  const int nxb = (C + 31) / 32;
  const bool is_x = (int)blockIdx.x < nxb;
  const int l0 = (is_x ? (int)blockIdx.x : (int)blockIdx.x - nxb) * 32;
  const int nl = is_x ? C : R;
  const int b0 = blockIdx.y * 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < 32) {
    const int b = b0 + threadIdx.x;
    if (b < B) {
      const double lrb = lr ? lr[b] : lr_scalar;
      plan[threadIdx.x] =
          make_plan(lrb, (double)xm[b], (double)dm[b], dwmin_b ? dwmin_b[b] : dw_min, BL, blm);
      if (blockIdx.x == 0 && bl_out) bl_out[b] = plan[threadIdx.x].skip ? 0 : plan[threadIdx.x].bl;
    }
  }
  __syncthreads();
  const int line = l0 + lane;
  const float *V = is_x ? X : D;
  // 4 words per thread (samples warp + 8 it), their Philox chains interleaved
  // call by call -- train_word's draws, in one loop, so the four dependent
  // chains overlap instead of running one word after the other
  const uint32_t lid = is_x ? (uint32_t)line : (uint32_t)(row0 + line);
  const uint32_t side = is_x ? 0u : 0x80000000u;
  uint32_t word[4], thr[4], c2[4], c3[4];
  int bl4[4], ng[4], gmax = 0;
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int s = warp + 8 * it;
    const int b = b0 + s;
    word[it] = thr[it] = c2[it] = c3[it] = 0u;
    bl4[it] = ng[it] = 0;
    if (b < B && line < nl) {
      const Plan pl = plan[s];
      const float v = V[(size_t)b * nl + line];
      if (!pl.skip) {
        double p = pl.amp * fabs((double)v) * (is_x ? pl.x_scale : pl.d_scale);
        p = (p < 1.0) ? p : 1.0;
        word[it] = v < 0.f ? 0x80000000u : 0u; // sign
        if (p >= 1.0) { // bernoulli(p >= 1) == 1, no draw
          word[it] |= (pl.bl >= 32) ? 0x7fffffffu : ((1u << pl.bl) - 1u);
        } else if (p > 0.0) {
          thr[it] = (uint32_t)(p * 4294967296.0); // P(u < thr) = thr / 2^32
          const uint64_t seq = seq0 + (uint64_t)b;
          c2[it] = (uint32_t)seq;
          c3[it] = (uint32_t)(seq >> 32) ^ side;
          bl4[it] = pl.bl;
          ng[it] = (pl.bl + 3) >> 2;
          gmax = max(gmax, ng[it]);
        }
      }
    }
  }
  for (int g = 0; g < gmax; ++g) {
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      if (g < ng[it]) {
        uint32_t a0 = (uint32_t)g, a1 = lid, a2 = c2[it], a3 = c3[it];
        philox10_rk(a0, a1, a2, a3, rk);
        uint32_t m = (uint32_t)(a0 < thr[it]) | ((uint32_t)(a1 < thr[it]) << 1) |
                     ((uint32_t)(a2 < thr[it]) << 2) | ((uint32_t)(a3 < thr[it]) << 3);
        const int rem = bl4[it] - 4 * g; // slots 4g .. 4g + 3 that exist
        if (rem < 4) m &= (1u << rem) - 1u;
        word[it] |= m << (4 * g);
      }
    }
  }
#pragma unroll
  for (int it = 0; it < 4; ++it) tile[lane][warp + 8 * it] = word[it];
  __syncthreads();
  if (is_x) { // quad layout (xq_index): thread = (column r, quad q), one uint4 store
    const int r = threadIdx.x & 31, q = threadIdx.x >> 5, ln = l0 + r, b = b0 + 4 * q;
    if (ln < nl && b < ldb)
      reinterpret_cast<uint4 *>(xw)[(size_t)(b >> 2) * C + ln] =
          make_uint4(tile[r][4 * q], tile[r][4 * q + 1], tile[r][4 * q + 2], tile[r][4 * q + 3]);
  } else {
    for (int r = warp; r < 32; r += 8) {
      const int ln = l0 + r, b = b0 + lane;
      if (ln < nl && b < B) dw[(size_t)ln * ldb + b] = tile[r][lane];
    }
  }
}

// deterministic_implicit needs the probabilities themselves: signed p
// (sign of the line, 0 for a no-op sample), sample-major [b][line]
__global__ void __launch_bounds__(256) probs_kernel(
    const float *__restrict__ X, const float *__restrict__ D, int C, int R,
    const double *__restrict__ lr, double lr_scalar, const float *__restrict__ xm,
    const float *__restrict__ dm, double dw_min, int BL, int blm, int32_t *__restrict__ bl_out,
    double *__restrict__ px, double *__restrict__ pd) {
  const int b = blockIdx.x;
  const Plan pl = make_plan(lr ? lr[b] : lr_scalar, (double)xm[b], (double)dm[b],
                            dw_min, BL, blm);
  if (threadIdx.x == 0 && bl_out) bl_out[b] = pl.skip ? 0 : pl.bl;
  for (int j = threadIdx.x; j < C; j += blockDim.x) {
    const float v = X[(size_t)b * C + j];
    double p = pl.amp * fabs((double)v) * pl.x_scale;
    p = (p < 1.0) ? p : 1.0;
    if (pl.skip) p = 0.0;
    px[(size_t)b * C + j] = (v < 0.f) ? -p : p;
  }
  for (int i = threadIdx.x; i < R; i += blockDim.x) {
    const float v = D[(size_t)b * R + i];
    double p = pl.amp * fabs((double)v) * pl.d_scale;
    p = (p < 1.0) ? p : 1.0;
    if (pl.skip) p = 0.0;
    pd[(size_t)b * R + i] = (v < 0.f) ? -p : p;
  }
}

void launch_trains(const Tile &t, const float *X, const float *D, int B, const double *lr_dev,
                   double lr_scalar, const float *xm, const float *dm, uint64_t seq0,
                   uint32_t *xw, uint32_t *dw, int ldb, int32_t *bl, double *px, double *pd,
                   bool deterministic, const double *dwmin_b) {
  if (B <= 0) return;
  if (deterministic) {
    probs_kernel<<<B, 256, 0, t.stream>>>(X, D, t.C, t.R, lr_dev, lr_scalar, xm, dm,
                                          t.cfg.device.dw_min, t.cfg.update.bl,
                                          t.cfg.update.bl_management, bl, px, pd);
  } else {
    dim3 grid((t.C + 31) / 32 + (t.R + 31) / 32, (B + 31) / 32);
    trains_kernel<<<grid, 256, 0, t.stream>>>(X, D, t.C, t.R, B, lr_dev, lr_scalar, xm, dm,
                                              t.cfg.device.dw_min, dwmin_b, t.cfg.update.bl,
                                              t.cfg.update.bl_management, round_keys(t.k_upd), seq0, t.row0,
                                              xw, dw, ldb, bl);
  }
  count_launch();
  XB_CUDA(cudaGetLastError());
}

// ============================================================== device laws
// proj/src/device.cpp:48-77; see WCell below for the per-pulse arithmetic.
struct LawArgs {
  float slope, gamma, std;
  float k2; // -2 ln2 std^2 (the angle table holds sqrt(-k2) (cos, sin))
  // upper bound of a c2c factor f = 1 + r t: r <= sqrt(17) (16-bit radius
  // uniform >= 2^-17), |t| <= sqrt(2 ln2) std, with a margin for the MUFU
  // approximations (the clamp-free SoftBounds pulses need f dw < |bound|)
  float fmax;
};

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}


__device__ __forceinline__ void box_muller_fast(uint32_t a, uint32_t b, float &z0, float &z1) {
  // u in (0, 1] and theta in [-pi, pi) straight from the mantissa bits
  const float u = 2.0f - __int_as_float(0x3f800000u | (a >> 9));
  const float th = fmaf(__int_as_float(0x3f800000u | (b >> 9)), 6.2831853071795865f,
                        -9.4247779607693797f);
  float l, r, s, c;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(u));
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(l * -1.3862943611198906f)); // -2 ln u
  asm("sin.approx.ftz.f32 %0, %1;" : "=f"(s) : "f"(th));
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(c) : "f"(th));
  z0 = r * c;
  z1 = r * s;
}

// c2c factors f = 1 + std z directly.  Box-Muller with the angle from a
// (cos, sin) table in shared memory (one LDS.64 instead of two MUFU ops) whose
// entries are pre-scaled by sqrt(2 ln2) std, so the radius is sqrt(-lg2 u)
// (the negation is a MUFU source modifier) and each factor one FMA, 1 + r cos.
// On a symmetric grid of >= 5 angles the moments E[cos^2] = 1/2, E[cos^4] =
// 3/8, E[cos^2 sin^2] = 1/8 are exact, so the factors keep unit variance, zero
// cross-correlation and Gaussian kurtosis.  Four pairs (8 factors) come from
// THREE Philox words -- 16-bit radius + 8-bit angle per pair -- so a 32-pulse
// stream word needs 3 Philox calls instead of 4.
// (an IMAD-only int->float variant measured 12 % slower: the XU has room for I2F)
constexpr int BM_ANGLES = 256; // (cos, sin) table entries in shared memory

// one pair from a 16-bit radius (as float) and an angle byte offset into the
// table (entries (cos, sin) * sqrt(2 ln2) std)
__device__ __forceinline__ void factor_pair_rt(float k16, uint32_t off,
                                               const float2 *__restrict__ cs, float &f0,
                                               float &f1) {
  const float u = fmaf(k16, 1.52587890625e-05f, 7.62939453125e-06f);
  float l, r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(u));
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(-l));
  const float2 t =
      *reinterpret_cast<const float2 *>(reinterpret_cast<const char *>(cs) + off);
  f0 = fmaf(r, t.x, 1.0f);
  f1 = fmaf(r, t.y, 1.0f);
}

// 8 factors from 3 words: radii a.hi, b.hi, c.hi, c.lo (I2F reads the halves in
// place); angles a.byte0, a.byte1, b.byte0, b.byte1 as byte offsets (x 8)
__device__ __forceinline__ void factor8_3w(uint32_t a, uint32_t b, uint32_t c,
                                           const float2 *__restrict__ cs, float *f) {
  factor_pair_rt((float)(a >> 16), (a << 3) & 0x7f8u, cs, f[0], f[1]);
  factor_pair_rt((float)(b >> 16), (a >> 5) & 0x7f8u, cs, f[2], f[3]);
  factor_pair_rt((float)(c >> 16), (b << 3) & 0x7f8u, cs, f[4], f[5]);
  factor_pair_rt((float)(unsigned short)c, (b >> 5) & 0x7f8u, cs, f[6], f[7]);
}



__device__ __forceinline__ void normal4_fast(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                             Key key, float &z0, float &z1, float &z2,
                                             float &z3) {
  philox10(c0, c1, c2, c3, key);
  box_muller_fast(c0, c1, z0, z1);
  box_muller_fast(c2, c3, z2, z3);
}

// ---- device laws for the pulse kernel, folded per (cell, direction) into
// affine constants (proj/src/device.cpp:51-76):
//   h  = step of this pulse, signed    ConstantStep  +dw_up | -dw_down
//                                      SoftBounds    dw_up - (dw_up/w_max) w | -dw_down + (dw_down/w_min) w
//                                      LinearStep    dw_up - dw_up slope w | -dw_down - dw_down slope w
//                                      ExpStep       dw_up 2^(-g (w - w_min)) | -dw_down 2^(-g (w_max - w))
//   w' = clamp(w + (1 + std z) h, w_min, w_max)
// so a pulse is two FMAs, a predicated select and two min/max (plus EX2 for
// ExpStep), all in fp32 on the stored weight.
template <int LAW> struct WCell {
  float wmin, wmax;
  float cu, cd; // constant parts (signed)
  float bu, bd; // slopes in w (ExpStep: exponent offsets)
  float g;      // ExpStep exponent scale gamma log2(e) / range

  __device__ __forceinline__ void init(float4 p, const LawArgs &la) {
    wmin = p.w;
    wmax = p.z;
    cu = p.x;
    cd = -p.y;
    bu = bd = g = 0.f;
    if (LAW == XB_SOFT_BOUNDS) {
      bu = -p.x / p.z;
      bd = p.y / p.w;
    } else if (LAW == XB_LINEAR_STEP) {
      bu = -p.x * la.slope;
      bd = -p.y * la.slope;
    } else if (LAW == XB_EXP_STEP) {
      g = la.gamma / (p.z - p.w) * 1.4426950408889634f;
      bu = g * p.w;  // up exponent  -g w + g w_min
      bd = -g * p.z; // down exponent g w - g w_max
    }
  }
  // one pulse; f = 1 + std z (1 without c2c noise).  CLAMP = false only where
  // the clamp is provably a no-op (see soft_bounds_clamp_free below).
  template <bool CLAMP = true>
  __device__ __forceinline__ float step(float w, float f, bool up) const {
    float h;
    if (LAW == XB_CONSTANT_STEP) {
      h = up ? cu : cd;
    } else if (LAW == XB_EXP_STEP) {
      const float e = up ? fmaf(-g, w, bu) : fmaf(g, w, bd);
      h = (up ? cu : cd) * ex2_approx(e);
    } else {
      const float hu = fmaf(bu, w, cu), hd = fmaf(bd, w, cd);
      h = up ? hu : hd;
    }
    const float wn = fmaf(f, h, w);
    return CLAMP ? fminf(fmaxf(wn, wmin), wmax) : wn;
  }
  // the same pulse on a compensated weight hi + lo: the law reads hi, the step
  // d = f h is added with an error-free two-sum, so the per-pulse rounding of
  // an fp32 add is carried in lo instead of accumulating (the reference keeps
  // fp64 weights; at dw_min = 1e-6 a step is only ~17 fp32 ulps of w = 0.5)
  __device__ __forceinline__ void step2(float &hi, float &lo, float f, bool up) const {
    float h;
    if (LAW == XB_CONSTANT_STEP) {
      h = up ? cu : cd;
    } else if (LAW == XB_EXP_STEP) {
      const float e = up ? fmaf(-g, hi, bu) : fmaf(g, hi, bd);
      h = (up ? cu : cd) * ex2_approx(e);
    } else {
      const float hu = fmaf(bu, hi, cu), hd = fmaf(bd, hi, cd);
      h = up ? hu : hd;
    }
    const float d = __fmul_rn(f, h);
    const float s = __fadd_rn(hi, d), bp = __fsub_rn(s, hi);
    const float e = __fadd_rn(__fsub_rn(hi, __fsub_rn(s, bp)), __fsub_rn(d, bp));
    const float c = fminf(fmaxf(s, wmin), wmax);
    lo = (c == s) ? __fadd_rn(lo, e) : 0.f;
    hi = c;
  }
};

// hi + lo -> (fl(hi + lo), exact residual): the stored hi is the best fp32
// weight (what the MVM and get_weights read), lo keeps the rest
__device__ __forceinline__ void renorm2(float &hi, float &lo) {
  const float s = __fadd_rn(hi, lo);
  lo = __fsub_rn(lo, __fsub_rn(s, hi));
  hi = s;
}

// ============================================================== K5: pulse
// One warp = one row i of the tile and 32 consecutive columns (one cell per
// lane); w and the cell's realization stay in registers for the whole batch.
// The batch is consumed in segments:
//   pre-pass (branch-free, sample order): per sample b, c = x_b & d_b (slot
//     bits), k = popc(c), direction = sign(x) * sign(d); the lane appends k
//     direction bits to its private pulse stream in shared memory
//     (1 = down, 0 = up).  A segment ends when some lane's stream would pass
//     CAP pulses (a warp vote), so any batch size and pulse density fit.
//   pulse loop: iteration n applies pulse n of every lane whose stream is
//     longer than n: the direction bit selects the law constants, the c2c
//     factors come from warp-uniform Philox refills (3 calls per 32 pulses).
// Lanes therefore wait only on the longest stream of the segment, and the
// per-cell pulse order is exactly the reference's (sample order; one
// direction per sample; pulses of a sample are interchangeable).
// The c2c normals of stream word m of a cell's segment come from
// Philox(k_c2c, (g0 + 3m + {0,1,2}, j, i, call)) with g0 the cell's running
// call count: independent of launch geometry and of row sharding.
// (56 x 32 lanes x 4 B x 32 warps = 224 KB: the segment capacity that still
// fits with the angle table; longer segments even out the lanes' stream
// lengths -- 5.55 -> 5.44 ms vs 32 words on the NS update)
#ifndef XB_PULSE_QW
#define XB_PULSE_QW 56
#endif
constexpr int PULSE_QW = XB_PULSE_QW;    // stream words per lane
constexpr int PULSE_CAP = PULSE_QW * 32; // pulses per lane per segment

// Launch shape (B200, round 1): persistent warps, ONE 1024-thread CTA per SM
// (64 registers; a few bytes spill outside the loops).  NS update: 7.48 ms vs 7.65 ms with two
// 512-thread CTAs and 8.0 ms with four 256-thread CTAs; ExpStep (cfg3):
// 13.5 ms vs 13.8 ms for a per-tile grid of 512-thread CTAs.
// (more warps at fewer registers lose: 2 CTAs x 18 or 20 warps, 56/51 regs,
// 6.89/6.91 ms vs 6.56 ms for 1 x 32 warps at 64 regs)
#ifndef XB_PULSE_WARPS
#define XB_PULSE_WARPS 32
#endif
#ifndef XB_PULSE_CTAS
#define XB_PULSE_CTAS 1
#endif
constexpr int PULSE_WARPS = XB_PULSE_WARPS;
// samples per vector block of the pre-pass (4: one uint4 of x and of d words;
// measured 6 % slower than 8)
#ifndef XB_PULSE_PB
#define XB_PULSE_PB 8
#endif

template <int LAW, bool NOISE, bool COMP>
__global__ void __launch_bounds__(PULSE_WARPS * 32, XB_PULSE_CTAS) pulse_kernel(
    float *__restrict__ W, float *__restrict__ Wlo, const float2 *__restrict__ S,
    const float2 *__restrict__ Bd, int ld, int R,
    int C,
    const uint32_t *__restrict__ xw, const uint32_t *__restrict__ dw, int ldb, int B, int row0,
    LawArgs la, RoundKeys rk, uint32_t call, uint32_t two, uint32_t flip,
    const int *__restrict__ abort_flag, uint32_t cb0, uint32_t ncb_run,
    unsigned *__restrict__ ctr) {
  extern __shared__ uint32_t qsm[]; // [PULSE_WARPS][PULSE_QW][32] streams, then the angle table
  if (abort_flag && *abort_flag) return; // rejected input: the tile stays untouched
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t *q = qsm + warp * (PULSE_QW * 32) + lane;
  float2 *cs = reinterpret_cast<float2 *>(qsm + PULSE_WARPS * PULSE_QW * 32);
  if (NOISE) {
    for (int k = threadIdx.x; k < BM_ANGLES; k += blockDim.x) {
      double sn, cn;
      sincospi((2.0 * k + 1.0) / BM_ANGLES, &sn, &cn); // (k + 1/2) 2 pi / BM_ANGLES
      const double r = sqrt(-(double)la.k2);               // sqrt(2 ln2) std
      cs[k] = make_float2((float)(cn * r), (float)(sn * r));
    }
    __syncthreads();
  }
  // persistent warps: each walks (row, 32-column block) items with a stride
  // of the whole grid, column-block major -- the warps of a CTA take
  // consecutive rows of ONE 32-column block, so they read the same x train
  // words (L1 hits) and the L2 sees each x word once per CTA, not per row.
  // Warps drift out of phase, so the ALU/FMA-bound pre-pass of some overlaps
  // the pulse loop of others.
  // items of the column blocks [cb0, cb0 + ncb_run) only (a one-hot x, e.g.
  // a Tiki-Taka transfer, has no coincidences anywhere else)
  // The last XB_PULSE_DYN_ROUNDS rounds are handed out from a work queue
  // instead (ctr[0]: next ticket): items differ in cost (the longest stream
  // of a row decides) and warps drift, so a static stride ends on its slowest
  // warps.  Measured on the NS update: 5.40 ms static, 5.32 with one queued
  // round, 5.27 with 4-16, 5.28 fully queued (the static part keeps the
  // CTA's warps on one column block).  The warp that retires last resets the
  // queue for the next launch on the stream.
  const uint32_t n_items = (uint32_t)R * ncb_run; // < 2^31 for any tile that fits
  const uint32_t nwarps = gridDim.x * PULSE_WARPS;
  const uint32_t rounds = n_items / nwarps;
#ifndef XB_PULSE_DYN_ROUNDS
#define XB_PULSE_DYN_ROUNDS 8
#endif
  const uint32_t dyn0 = (rounds > XB_PULSE_DYN_ROUNDS ? rounds - XB_PULSE_DYN_ROUNDS : 0) * nwarps;
  uint32_t item = blockIdx.x * PULSE_WARPS + warp;
  for (;;) {
    if (item >= dyn0) { // queued part: one ticket per warp per item
      uint32_t tk = 0;
      if (lane == 0) tk = atomicAdd(ctr, 1u);
      item = dyn0 + __shfl_sync(0xffffffffu, tk, 0);
    }
    if (item >= n_items) {
      if (lane == 0 && atomicAdd(ctr + 1, 1u) == nwarps - 1) {
        ctr[0] = 0u; // every warp has drawn its last ticket: reset for the next launch
        ctr[1] = 0u;
      }
      break;
    }
    {
  const uint32_t cb = cb0 + item / (uint32_t)R;
  const int i = (int)(item - (cb - cb0) * (uint32_t)R);
  const int j = (int)cb * 32 + lane;
  const bool valid = j < C;
  const size_t idx = (size_t)i * ld + j;

  float w = 0.f, wlo = 0.f; // wlo: compensation term (COMP)
  WCell<LAW> cell;
  float4 pc = make_float4(0.f, 0.f, 1.f, -1.f);
  if (valid) {
    const float2 st = S[idx], bd = Bd[idx];
    pc = make_float4(st.x, st.y, bd.x, bd.y);
  }
  cell.init(pc, la);
#ifdef XB_SB_ALWAYS_CLAMP
  constexpr bool SB_FREE = false; // experiment build: the clamp on every pulse
#else
  constexpr bool SB_FREE = LAW == XB_SOFT_BOUNDS && !COMP;
#endif
  // clamp-free SoftBounds pulses (apply8) need f dw < |bound| in every cell of
  // the warp: a realized cell with an extreme dw / bound ratio (d2d floors)
  // keeps its item on the clamped path
  const bool item_free =
      SB_FREE && __all_sync(0xffffffffu, la.fmax * pc.x <= pc.z && la.fmax * pc.y <= -pc.w);
  if (valid) w = W[idx];
  if (COMP && valid) wlo = Wlo[idx];
  const uint32_t jg = (uint32_t)j, ig = (uint32_t)(row0 + i);
  // this lane's x words (quad layout: 4 samples per uint4, stride C uint4s)
  // and the warp's d line (line-major, ldb % 8 == 0)
  const uint4 *xq = reinterpret_cast<const uint4 *>(xw) + (valid ? j : 0);
  const uint32_t *dline = dw + (size_t)i * ldb;
  const uint32_t xmask = valid ? 0x7fffffffu : 0u; // idle lanes see no coincidences
  const uint32_t q0 = (uint32_t)__cvta_generic_to_shared(q);
  uint32_t g0 = 0;

  int b = 0;
  while (b < B) {
    // ---------------- pre-pass: append this lane's pulses, sample order.
    // sh = fill of the open stream word acc, qa = its shared address; the
    // stream length is T = (qa - q0) / 4 + sh (32 pulses per 128-B word step).
    uint32_t sh = 0, acc = 0, qa = q0;
    // The pulse direction is bit 31 of x ^ d ^ flip (the line signs); it is
    // moved to bit 0 with a multiply-high on the FMA pipe (dn = 1 iff down)
    // and the stream bits (1 = down) are added with a multiply-add (the bits
    // are disjoint), which balances the pre-pass between the ALU and FMA pipes
    auto append = [&](uint32_t xv, uint32_t dv) {
      const uint32_t k = __popc(xv & dv & xmask);
      uint32_t dn, lo;
      asm("mul.hi.u32 %0, %1, %2;" : "=r"(dn) : "r"(xv ^ dv ^ flip), "r"(two));
      asm("bmsk.clamp.b32 %0, %1, %2;" : "=r"(lo) : "r"(sh), "r"(k)); // k ones from bit sh
      asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(acc) : "r"(lo), "r"(dn));
      uint32_t e = sh + k;
      if (e >= 32u) {
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(qa), "r"(acc));
        qa += 128u;
        e -= 32u; // e < 63: a predicated add (FMA pipe) instead of an AND (ALU)
        uint32_t hi;
        asm("bmsk.clamp.b32 %0, %1, %2;" : "=r"(hi) : "r"(0u), "r"(e));
        asm("mul.lo.u32 %0, %1, %2;" : "=r"(acc) : "r"(hi), "r"(dn));
      }
      sh = e;
    };
    auto stream_len = [&]() { return ((qa - q0) >> 2) + sh; };
    // fast path: aligned blocks of PB samples held as NV uint4 slots of x
    // and of d words; each slot is refilled with the next block's words as
    // soon as it is consumed (rolling prefetch, no register copies).  A block
    // is taken only if it cannot overflow any lane's stream.
    constexpr int PB = XB_PULSE_PB, NV = PB / 4;
    if ((b % PB) == 0 && b + PB <= B) {
      // running pointers: one 64-bit step per block instead of index math
      const uint4 *xn = xq + (size_t)(b >> 2) * C;
      const uint4 *dn = reinterpret_cast<const uint4 *>(dline) + (b >> 2);
      const size_t xs = (size_t)C * NV; // uint4s per block of x
      uint4 xa[NV], da[NV];
#pragma unroll
      for (int u = 0; u < NV; ++u) {
        xa[u] = __ldg(xn + (size_t)u * C);
        da[u] = __ldg(dn + u);
      }
      // a block adds at most PB * 31 pulses to a lane's stream: `room` is a
      // warp-uniform lower bound on the space left, refreshed by a max
      // reduction only when it could not take another block
      uint32_t room = 0;
      while (true) {
        if (room < PB * 31u) {
          room = (uint32_t)PULSE_CAP - __reduce_max_sync(0xffffffffu, stream_len());
          if (room < PB * 31u) break;
        }
        room -= PB * 31u;
        const int bn = b + PB;
        const bool more = bn + PB <= B;
        xn += xs;
        dn += NV;
#pragma unroll
        for (int u = 0; u < NV; ++u) {
          append(xa[u].x, da[u].x);
          append(xa[u].y, da[u].y);
          append(xa[u].z, da[u].z);
          append(xa[u].w, da[u].w);
          if (more) {
            xa[u] = __ldg(xn + (size_t)u * C);
            da[u] = __ldg(dn + u);
          }
        }
        b = bn;
        if (!more) break;
      }
    }
    // careful path, one sample at a time: the batch tail, or a stream near CAP
    while (b < B) {
      const uint32_t xv = __ldg(reinterpret_cast<const uint32_t *>(xq + (size_t)(b >> 2) * C) +
                                (b & 3)),
                     dv = __ldg(dline + b);
      if (__any_sync(0xffffffffu, stream_len() + __popc(xv & dv & xmask) > (uint32_t)PULSE_CAP))
        break;
      append(xv, dv);
      ++b;
    }
    if (sh) asm volatile("st.shared.u32 [%0], %1;" ::"r"(qa), "r"(acc));
    const uint32_t T = stream_len();
    const uint32_t minT = __reduce_min_sync(0xffffffffu, T);
    const uint32_t maxT = __reduce_max_sync(0xffffffffu, T);
    __syncwarp();

    // ---------------- pulse loop: pulse n of every lane with n < T.  Words
    // below the shortest stream need no per-pulse activity test.
    // check: vm holds this lane's valid-pulse bits of the word (a prefix),
    // tested like the direction bits instead of comparing n + v with T
    // SoftBounds without a negative c2c factor never leaves [w_min, w_max]:
    // an up pulse gives w' - w_max = (w - w_max)(1 - f dw_up / w_max) <= 0 and
    // w' >= w for 0 <= f < w_max / dw_up (the fp32 evaluation keeps both: h
    // carries the factor (w_max - w) exactly up to a relative rounding, and
    // fp32 rounding is monotone, so fl(w') never crosses a representable
    // bound); down pulses mirror it.  So the two-sided clamp of
    // proj/src/device.cpp:76 is a no-op there and is skipped: the 8 factors
    // of a block are tested for a sign bit (3 LOP3 + a vote), and only a warp
    // holding a negative factor (~10 % of blocks at std 0.3) runs the
    // clamped pulses.  The weights are bit-identical either way.
    auto apply8 = [&](uint32_t word, int sh8, bool check, uint32_t vm, const float *f) {
      bool clamp = true;
      if (SB_FREE && item_free) {
        if (!NOISE) {
          clamp = false; // f = 1
        } else {
          const uint32_t neg = __float_as_uint(f[0]) | __float_as_uint(f[1]) |
                               __float_as_uint(f[2]) | __float_as_uint(f[3]) |
                               __float_as_uint(f[4]) | __float_as_uint(f[5]) |
                               __float_as_uint(f[6]) | __float_as_uint(f[7]);
          clamp = __any_sync(0xffffffffu, (int)neg < 0);
        }
      }
      if (SB_FREE && !clamp) {
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const float wn = cell.template step<false>(w, f[v], ((word >> (sh8 + v)) & 1u) == 0u);
          if (!check || ((vm >> (sh8 + v)) & 1u)) w = wn;
        }
        return;
      }
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        if (COMP) {
          float hn = w, ln = wlo;
          cell.step2(hn, ln, f[v], ((word >> (sh8 + v)) & 1u) == 0u);
          if (!check || ((vm >> (sh8 + v)) & 1u)) {
            w = hn;
            wlo = ln;
          }
        } else {
          const float wn = cell.step(w, f[v], ((word >> (sh8 + v)) & 1u) == 0u);
          if (!check || ((vm >> (sh8 + v)) & 1u)) w = wn;
        }
      }
      // keep lo below an ulp of hi: its own rounding then stays negligible
      // (left to grow, lo collects a systematic error of its own)
      if (COMP) renorm2(w, wlo);
    };
    // one 32-pulse stream word: Philox calls g0 + 3 m + {0, 1, 2} (m = word
    // index) give 12 words, three per 8-pulse block; `lim` (warp-uniform)
    // cuts the ragged last word
    auto word32 = [&](uint32_t word, uint32_t n0, bool check, uint32_t vm, uint32_t lim) {
      float f[8] = {1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f};
      uint32_t p0 = 0, p1 = 0, p2 = 0, p3 = 0, r0 = 0, r1 = 0, r2 = 0, r3 = 0;
      const uint32_t base = g0 + 3u * (n0 >> 5);
      if (NOISE) {
        p0 = base, p1 = jg, p2 = ig, p3 = call;
        philox10_rk<XB_C2C_ROUNDS>(p0, p1, p2, p3, rk);
        factor8_3w(p0, p1, p2, cs, f);
      }
      apply8(word, 0, check, vm, f);
      if (lim <= 8u) return;
      if (NOISE) {
        r0 = base + 1u, r1 = jg, r2 = ig, r3 = call;
        philox10_rk<XB_C2C_ROUNDS>(r0, r1, r2, r3, rk);
        factor8_3w(p3, r0, r1, cs, f);
      }
      apply8(word, 8, check, vm, f);
      if (lim <= 16u) return;
      if (NOISE) {
        p0 = base + 2u, p1 = jg, p2 = ig, p3 = call;
        philox10_rk<XB_C2C_ROUNDS>(p0, p1, p2, p3, rk);
        factor8_3w(r2, r3, p0, cs, f);
      }
      apply8(word, 16, check, vm, f);
      if (lim <= 24u) return;
      if (NOISE) factor8_3w(p1, p2, p3, cs, f);
      apply8(word, 24, check, vm, f);
    };
    uint32_t n0 = 0;
    for (; n0 + 32u <= minT; n0 += 32u) word32(q[(n0 >> 5) * 32], n0, false, 0u, 32u);
    for (; n0 < maxT; n0 += 32u) {
      uint32_t vm; // bits [0, T - n0) of this word are pulses of this lane
      asm("bmsk.clamp.b32 %0, %1, %2;" : "=r"(vm) : "r"(0u), "r"(T > n0 ? T - n0 : 0u));
      word32(q[(n0 >> 5) * 32], n0, true, vm, maxT - n0);
    }
    g0 += 3u * ((T + 31u) >> 5);
    __syncwarp();
  }
  if (COMP) renorm2(w, wlo);
  if (valid) W[idx] = w;
  if (COMP && valid) Wlo[idx] = wlo;
    }
    item += nwarps; // static part: stride of the whole grid
  }
}

template <int LAW, bool NOISE, bool COMP>
static void pulse_dispatch(Tile &t, const uint32_t *xw, const uint32_t *dw, int ldb, int B,
                           LawArgs la, uint32_t call, bool flip, int col) {
  const int smem = PULSE_WARPS * PULSE_QW * 32 * (int)sizeof(uint32_t) +
                   (NOISE ? BM_ANGLES * (int)sizeof(float2) : 0);
  // persistent grid: every resident CTA slot of the device, capped by the work
  static std::atomic<uint64_t> configured{0};
  static std::atomic<int> blocks_of[64];
  once_per_device(configured, [&] {
    XB_CUDA(cudaFuncSetAttribute(pulse_kernel<LAW, NOISE, COMP>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int per_sm = 0, sms = 0;
    XB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pulse_kernel<LAW, NOISE, COMP>,
                                                          PULSE_WARPS * 32, smem));
    XB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, current_device()));
    blocks_of[current_device() & 63].store(std::max(1, per_sm) * sms);
  });
  const int blocks = blocks_of[current_device() & 63].load();
  const uint32_t cb0 = col >= 0 ? (uint32_t)(col / 32) : 0u;
  const uint32_t ncb_run = col >= 0 ? 1u : (uint32_t)((t.C + 31) / 32);
  const long items = (long)t.R * ncb_run;
  const dim3 grid((unsigned)std::min<long>(blocks, (items + PULSE_WARPS - 1) / PULSE_WARPS));
  if (!t.pulse_ctr) {
    XB_CUDA(cudaMalloc(&t.pulse_ctr, 2 * sizeof(unsigned)));
    XB_CUDA(cudaMemsetAsync(t.pulse_ctr, 0, 2 * sizeof(unsigned), t.stream));
  }
  pulse_kernel<LAW, NOISE, COMP><<<grid, PULSE_WARPS * 32, smem, t.stream>>>(
      t.W, t.Wlo, t.steps(), t.bounds(), t.ld, t.R, t.C, xw, dw, ldb, B, t.row0, la,
      round_keys(t.k_c2c), call, 2u,
      flip ? 0x80000000u : 0u, t.abort_flag, cb0, ncb_run, t.pulse_ctr);
  count_launch();
  XB_CUDA(cudaGetLastError());
}

void launch_pulse(Tile &t, const uint32_t *xw, const uint32_t *dw, int ldb, int B,
                  uint32_t call_id, bool flip, int col) {
  if (B <= 0 || t.R == 0) return;
  const double sd = t.cfg.device.dw_min_std;
  const LawArgs la{(float)t.cfg.device.slope, (float)t.cfg.device.gamma, (float)sd,
                   (float)(-2.0 * 0.6931471805599453 * sd * sd), (float)(1.0 + 5.0 * sd + 1e-3)};
  const bool noise = t.cfg.device.dw_min_std > 0.0;
#define XB_PULSE(K)                                                                        \
  case K:                                                                                  \
    if (t.comp)                                                                            \
      noise ? pulse_dispatch<K, true, true>(t, xw, dw, ldb, B, la, call_id, flip, col)          \
            : pulse_dispatch<K, false, true>(t, xw, dw, ldb, B, la, call_id, flip, col);        \
    else                                                                                   \
      noise ? pulse_dispatch<K, true, false>(t, xw, dw, ldb, B, la, call_id, flip, col)         \
            : pulse_dispatch<K, false, false>(t, xw, dw, ldb, B, la, call_id, flip, col);       \
    break;
  switch (t.cfg.device.kind) {
    XB_PULSE(XB_CONSTANT_STEP)
    XB_PULSE(XB_LINEAR_STEP)
    XB_PULSE(XB_SOFT_BOUNDS)
    XB_PULSE(XB_EXP_STEP)
  default:
    raise("device.kind: unknown device model");
  }
#undef XB_PULSE
}

// ============================================================== sample gather
// out[line][k] = in[line][idx[k]] for k < n, zero up to ldb_out: the trains of
// the samples one unit-cell member receives (round-robin policy)
__global__ void gather_samples_kernel(const uint32_t *__restrict__ in, int ldb_in, int lines,
                                      const int *__restrict__ idx, int n,
                                      uint32_t *__restrict__ out, int ldb_out, bool quad) {
  for (int line = blockIdx.y; line < lines; line += gridDim.y) // (gridDim.y <= 65535)
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < ldb_out; k += gridDim.x * blockDim.x) {
      if (quad)
        out[xq_index(line, k, lines)] = k < n ? in[xq_index(line, idx[k], lines)] : 0u;
      else
        out[(size_t)line * ldb_out + k] = k < n ? in[(size_t)line * ldb_in + idx[k]] : 0u;
    }
}

void launch_gather_samples(const uint32_t *in, int ldb_in, int lines, const int *idx, int n,
                           uint32_t *out, int ldb_out, cudaStream_t s, bool quad) {
  if (lines <= 0 || ldb_out <= 0) return;
  const int threads = std::min(256, (ldb_out + 31) / 32 * 32);
  dim3 grid((ldb_out + threads - 1) / threads, std::min(lines, 65535));
  gather_samples_kernel<<<grid, threads, 0, s>>>(in, ldb_in, lines, idx, n, out, ldb_out, quad);
  count_launch();
  XB_CUDA(cudaGetLastError());
}

// ============================================================== K6: deterministic
// proj/src/pulsed.cpp:128-144: count = lround(bl * p_d * p_x) in fp64, pulses
// in one direction per (cell, sample).  Signed probabilities carry the line
// signs (p = 0 <=> sign 0 or a no-op sample).
template <int LAW, bool NOISE, bool COMP>
__global__ void __launch_bounds__(256) pulse_det_kernel(
    float *__restrict__ W, float *__restrict__ Wlo, const float2 *__restrict__ S,
    const float2 *__restrict__ Bd, int ld, int R,
    int C, const double *__restrict__ px, const double *__restrict__ pd,
    const int32_t *__restrict__ bl, int B, int row0, LawArgs la, Key key, uint32_t call,
    const int *__restrict__ abort_flag) {
  if (abort_flag && *abort_flag) return; // rejected input: the tile stays untouched
  const int j = blockIdx.x * 32 + (threadIdx.x & 31);
  const int i = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (i >= R || j >= C) return;
  const size_t idx = (size_t)i * ld + j;
  float w = W[idx], wlo = COMP ? Wlo[idx] : 0.f;
  WCell<LAW> cell;
  cell.init(make_float4(S[idx].x, S[idx].y, Bd[idx].x, Bd[idx].y), la);
  uint32_t n = 0;
  float z[4] = {0.f, 0.f, 0.f, 0.f};
  for (int b = 0; b < B; ++b) {
    const double a = pd[(size_t)b * R + i], x = px[(size_t)b * C + j];
    if (a == 0.0 || x == 0.0) continue;
    const long long count = llround((double)bl[b] * fabs(a) * fabs(x));
    const bool up = (a > 0.0) == (x > 0.0);
    for (long long k = 0; k < count; ++k, ++n) {
      if (NOISE && (n & 3u) == 0u)
        normal4_fast(n >> 2, (uint32_t)j, (uint32_t)(row0 + i), call, key, z[0], z[1], z[2], z[3]);
      const float f = NOISE ? fmaf(la.std, z[n & 3u], 1.0f) : 1.0f;
      if (COMP) {
        cell.step2(w, wlo, f, up);
        renorm2(w, wlo);
      } else {
        w = cell.step(w, f, up);
      }
    }
  }
  if (COMP) {
    renorm2(w, wlo);
    Wlo[idx] = wlo;
  }
  W[idx] = w;
}

template <int LAW, bool NOISE, bool COMP>
static void det_dispatch(Tile &t, const double *px, const double *pd, const int32_t *bl, int B,
                         LawArgs la, uint32_t call) {
  dim3 grid((t.C + 31) / 32, (t.R + 7) / 8);
  pulse_det_kernel<LAW, NOISE, COMP><<<grid, 256, 0, t.stream>>>(
      t.W, t.Wlo, t.steps(), t.bounds(), t.ld, t.R, t.C, px, pd, bl, B, t.row0, la, t.k_c2c, call,
      t.abort_flag);
  count_launch();
  XB_CUDA(cudaGetLastError());
}

void launch_pulse_det(Tile &t, const double *px, const double *pd, const int32_t *bl, int B,
                      uint32_t call_id) {
  if (B <= 0 || t.R == 0) return;
  const double sd = t.cfg.device.dw_min_std;
  const LawArgs la{(float)t.cfg.device.slope, (float)t.cfg.device.gamma, (float)sd,
                   (float)(-2.0 * 0.6931471805599453 * sd * sd), (float)(1.0 + 5.0 * sd + 1e-3)};
  const bool noise = t.cfg.device.dw_min_std > 0.0;
#define XB_DET(K)                                                                          \
  case K:                                                                                  \
    if (t.comp)                                                                            \
      noise ? det_dispatch<K, true, true>(t, px, pd, bl, B, la, call_id)                   \
            : det_dispatch<K, false, true>(t, px, pd, bl, B, la, call_id);                 \
    else                                                                                   \
      noise ? det_dispatch<K, true, false>(t, px, pd, bl, B, la, call_id)                  \
            : det_dispatch<K, false, false>(t, px, pd, bl, B, la, call_id);                \
    break;
  switch (t.cfg.device.kind) {
    XB_DET(XB_CONSTANT_STEP)
    XB_DET(XB_LINEAR_STEP)
    XB_DET(XB_SOFT_BOUNDS)
    XB_DET(XB_EXP_STEP)
  default:
    raise("device.kind: unknown device model");
  }
#undef XB_DET
}

} // namespace xb
