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

// stores the outputs 4g..4g+3 that fall in [o0, o0 + M): one 16-byte store
// when the group is whole and aligned, else per element
__device__ __forceinline__ void store_group4(const float y[4], int g, int o0, int M,
                                             float *__restrict__ yrow) {
  const int o = 4 * g - o0;
  if (o >= 0 && o + 3 < M && ((reinterpret_cast<uintptr_t>(yrow + o) & 15u) == 0)) {
    *reinterpret_cast<float4 *>(yrow + o) = make_float4(y[0], y[1], y[2], y[3]);
    return;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (o + k >= 0 && o + k < M) yrow[o + k] = y[k];
}

// Outputs 4g..4g+3 (global index) of one sample: a[k] = their contraction
// sums; the ones inside [o0, o0 + M) are written to yrow[o - o0].  Returns
// whether any of them reached the ADC bound (bound management).
// the output values y[k] of outputs 4g + k (the store is the caller's)
__device__ __forceinline__ bool epilogue_values4(const float a[4], int g, int o0, int M,
                                                 const SampleState &s, const IoDev &io, Key key,
                                                 uint64_t seq, float y[4]) {
  bool hit = false;
  if (io.perfect) {
#pragma unroll
    for (int k = 0; k < 4; ++k) y[k] = a[k];
    return false;
  }
  uint32_t w[4] = {0u, 0u, 0u, 0u};
  const bool noisy = io.sigma_w > 0.0 || io.sigma_out > 0.0;
  if (noisy) out_noise_words((uint32_t)g, seq, s.m, key, w);
  if (!io.exact) {
    // fp32 output stage (tensor-core modes): alpha 2^m y rounds once in fp32,
    // exactly like the fp64 product cast to fp32 (2^m is exact)
    const float scale = s.alpha == 0.f ? 1.f : s.alpha * (float)pow2i(s.m);
    const float sw = (float)io.sigma_w * s.norm, so = (float)io.sigma_out;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float z0 = 0.f, z1 = 0.f;
      if (noisy) box_muller16(w[k], z0, z1);
      float v;
      if (s.alpha == 0.f) {
        v = so * z1;
      } else {
        v = a[k];
        if (io.sigma_w > 0.0) v = fmaf(sw, z0, v);
        v = fmaf(so, z1, v);
        // only outputs of this tile/shard count (a group may straddle its edge)
        const int o = 4 * g + k - o0;
        hit |= (o >= 0 && o < M) && fabsf(v) >= io.adc.fbound;
      }
      y[k] = scale * quantize_f(v, io.adc);
    }
    return hit;
  }
  const double scale = s.alpha == 0.f ? 1.0 : (double)s.alpha * pow2i(s.m);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float z0 = 0.f, z1 = 0.f;
    if (noisy) box_muller16(w[k], z0, z1);
    double v;
    if (s.alpha == 0.f) {
      v = io.sigma_out > 0.0 ? io.sigma_out * (double)z1 : 0.0;
    } else {
      v = (double)a[k];
      if (io.sigma_w > 0.0) v += io.sigma_w * (double)s.norm * (double)z0;
      if (io.sigma_out > 0.0) v += io.sigma_out * (double)z1;
      const int o = 4 * g + k - o0;
      hit |= (o >= 0 && o < M) && fabs(v) >= io.adc.bound;
    }
    y[k] = (float)(scale * quantize(v, io.adc));
  }
  return hit;
}

__device__ __forceinline__ bool epilogue_group4(const float a[4], int g, int o0, int M,
                                                const SampleState &s, const IoDev &io, Key key,
                                                uint64_t seq, float *__restrict__ yrow) {
  float y[4];
  const bool hit = epilogue_values4(a, g, o0, M, s, io, key, seq, y);
  store_group4(y, g, o0, M, yrow);
  return hit;
}

// BM bookkeeping: one flag store per warp (a saturating sample saturates many
// outputs).  A plain store of 1, never read back here: every writer stores the
// same value, and the readers run after a kernel boundary or a grid barrier
// (a returning atomic here would hold the warp for an L2 round trip per
// output column).  flag = this sample's word in the pass's flag array.
__device__ __forceinline__ void bm_flag(bool hit, const SampleState &s, const IoDev &io,
                                        int *flag) {
  if (io.bm && s.alpha != 0.f && s.m < io.bm_max_iter) {
    const unsigned any = __ballot_sync(__activemask(), hit);
    if (hit && (threadIdx.x & 31) == __ffs(any) - 1) *reinterpret_cast<volatile int *>(flag) = 1;
  }
}

// Bound-management bookkeeping, per N slab of nb samples (slab-local sample
// index b - n0):  pass p writes its saturation flags to flags[(p & 1) nb ..];
// the re-issue of pass p + 1 takes the flagged samples of pass p (ascending
// order, compacted -- their number lands in counts[32 + p] on the
// host-driven route), and clears the other parity's flags for pass p + 1.
// words per N slab (<= 256 samples): flags [2][256], counts [64]
constexpr int BM_SLAB_WORDS = 2 * 256 + 64;
struct BmBufs {
  int *flags;  // [2][nb]
  int *counts; // [64]; [32 + p]: compacted count for pass p (host-driven rounds)
  int *map;    // [nb] compacted sample list (global sample index)
};

// (x~ prep, one sample) proj/src/io.cpp:117-131: x~_j = Q_dac(x_j / (alpha 2^m))
// + sigma_inp xi_j in fp64 converter arithmetic.
struct RowDac {
  double inv;
  float a32, c032, tie_eps;
  bool fast;
  __device__ __forceinline__ RowDac(const SampleState &s, const IoDev &io) {
    inv = (s.alpha == 0.f) ? 0.0 : 1.0 / ((double)s.alpha * pow2i(s.m));
    // fp32 fast path of the DAC, bit-identical to the fp64 quantizer: the grid
    // index is k = round_half_away(t), t = x inv L / (2 b) + (L - 1) / 2
    // (L = 2^bits).  In fp32, t carries at most L 2^-23 of error; outside a
    // window of L 2^-20 around a half-integer both evaluations round the same
    // way, and inside it (rare) the element takes the fp64 path.  Without it
    // the DAC was fp64-conversion bound (~4 us per 4096-wide sample on B200).
    fast = !io.perfect && s.alpha != 0.f && io.dac.bits > 0 && io.dac.bits <= 16 && io.dac.pow2 &&
           io.sigma_inp == 0.0;
    a32 = fast ? (float)(inv * pow2i(io.dac.bits) / (2.0 * io.dac.bound)) : 0.f;
    c032 = 0.5f * (io.dac.flevels_m1); // (L - 1) / 2, exact
    tie_eps = fast ? __int_as_float((127 + io.dac.bits - 20) << 23) /* 2^(bits-20) */ : 0.f;
  }
  __device__ __forceinline__ float operator()(float xv, int j, const SampleState &s,
                                              const IoDev &io, Key key, uint64_t seq,
                                              int in0) const {
    if (io.perfect) return xv;
    if (s.alpha == 0.f) return 0.f;
    if (fast) {
      if (xv == 0.f) return 0.f; // exact zero passes (io.cpp:44)
      const float t = fmaf(xv, a32, c032);
      const float fr = t - floorf(t);
      if (fabsf(fr - 0.5f) > tie_eps) {
        float k = floorf(t + 0.5f); // not a tie: round-half-away == round-half-up here
        k = fminf(fmaxf(k, 0.f), io.dac.flevels_m1);
        return fmaf(k + 0.5f, io.dac.fstep, -io.dac.fbound);
      }
    }
    double q = quantize((double)xv * inv, io.dac);
    if (io.sigma_inp > 0.0) {
      const float z = normal1((uint32_t)(j + in0), (uint32_t)seq,
                              (uint32_t)(seq >> 32) | ((uint32_t)s.m << 24), TAG_IN_NOISE << 24,
                              key);
      q += io.sigma_inp * (double)z;
    }
    return (float)q;
  }
};

// ||x~|| from every thread's partial sum of squares: warp sums, then the
// warps in order (the order every x~ prep of the library shares)
__device__ __forceinline__ float row_norm(float nrm, float *red) {
  nrm = warp_sum(nrm);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nrm;
  __syncthreads();
  float tot = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
  __syncthreads();
  return sqrtf(tot);
}

// block size of every x~ prep (prep / re-issue kernels, the in-kernel loop):
// ||x~|| sums per-thread partials in this layout, so it fixes the bits
#define XB_PREP_THREADS 512

// the register path of the prep: element j = threadIdx.x + u blockDim.x is
// v[u] (n <= blockDim.x PREP_VPT); ||x~|| returned in every thread
constexpr int PREP_VPT = 8;
__device__ __forceinline__ float prep_row_vals(const float (&v)[PREP_VPT], int n,
                                               float *__restrict__ xt, const SampleState &s,
                                               const IoDev &io, Key key, uint64_t seq, int in0,
                                               float *red) {
  const RowDac dac(s, io);
  float nrm = 0.f;
#pragma unroll
  for (int u = 0; u < PREP_VPT; ++u) {
    const int j = threadIdx.x + u * (int)blockDim.x;
    if (j < n) {
      const float f = dac(v[u], j, s, io, key, seq, in0);
      xt[j] = f;
      nrm = fmaf(f, f, nrm);
    }
  }
  return row_norm(nrm, red);
}

// x~ row of one sample at level s.m, ||x~|| returned in every thread.  All
// threads of the block take part; red: >= 33 floats of shared.
__device__ __forceinline__ float prep_row(const float *__restrict__ x, int n,
                                          float *__restrict__ xt, const SampleState &s,
                                          const IoDev &io, Key key, uint64_t seq, int in0,
                                          float *red) {
  if (n <= (int)blockDim.x * PREP_VPT) { // all loads of a thread in flight first
    float v[PREP_VPT];
#pragma unroll
    for (int u = 0; u < PREP_VPT; ++u) {
      const int j = threadIdx.x + u * (int)blockDim.x;
      v[u] = j < n ? x[j] : 0.f;
    }
    return prep_row_vals(v, n, xt, s, io, key, seq, in0, red);
  }
  const RowDac dac(s, io);
  float nrm = 0.f;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const float f = dac(x[j], j, s, io, key, seq, in0);
    xt[j] = f;
    nrm = fmaf(f, f, nrm);
  }
  return row_norm(nrm, red);
}

// Block-wide compaction: map[0..n) = the indices i < nb with flags[i] != 0,
// ascending, written as base + i; returns n in every thread.  cnt: >= 33 ints
// of shared memory.
__device__ __forceinline__ int block_compact(const int *__restrict__ flags, int nb, int base,
                                             int *__restrict__ map, int *cnt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int total = 0;
  for (int i0 = 0; i0 < nb; i0 += blockDim.x) {
    const int i = i0 + threadIdx.x;
    const bool f = i < nb && flags[i] != 0;
    const unsigned m = __ballot_sync(0xffffffffu, f);
    if (lane == 0) cnt[warp] = __popc(m);
    __syncthreads();
    int before = 0, all = 0;
    for (int w = 0; w < nw; ++w) {
      before += (w < warp) ? cnt[w] : 0;
      all += cnt[w];
    }
    if (f) map[total + before + __popc(m & ((1u << lane) - 1u))] = base + i;
    total += all;
    __syncthreads();
  }
  return total;
}

// Grid-wide barrier of a launch whose CTAs are all co-resident (checked on
// the host with cudaOccupancyMaxActiveClusters): `target` = arrivals expected
// so far (k-th barrier: k * gridDim).  Release/acquire at gpu scope; a spin
// past ~2 s traps (a kernel error, never a hung GPU).
__device__ __forceinline__ void grid_sync(unsigned *ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    const long long t0 = clock64();
    unsigned v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      if (v >= target) break;
      if (clock64() - t0 > (1ll << 32)) __trap();
      __nanosleep(32);
    }
  }
  __syncthreads();
}

// arguments of the fused output stage (and of the in-kernel re-issue rounds)
struct FusedOut {
  float *Y;            // [B][ldy]
  int ldy;
  SampleState *st;     // per sample (global index)
  IoDev io;
  Key key;
  uint64_t seq0;       // sequence number of sample 0 of the call
  BmBufs bm;           // flags/counts/map of this N slab
  int pass;            // pass index of the launch's first pass (0, or a host-driven re-issue)
  int o0;              // global index of output 0 (row shards: row0; backward: 0)
  int n0;              // first sample (= x~ row of pass 0) of this N slab
  int nb;              // samples in this N slab
  const int *n_dev;    // host-driven re-issue: number of compacted samples (device), else null
  // in-kernel bound management (loop != 0): re-issue rounds inside this launch
  int loop;
  const float *X;      // raw inputs [B][K] (re-issue prep)
  int K, in0;          // input length; global index of input 0
  float *xt;           // x~ rows of this slab; re-issue rows are compacted from row 0
  int ldt;
  unsigned *bar;       // grid-barrier counter, zero at launch
  // x~ of every sample of the slab at m = 1, prepared during pass 0 by the
  // contraction's idle warps, and its states (global index): the first re-issue
  // streams this slab whole -- no compaction, prep or second barrier -- and
  // writes only the samples pass 0 flagged.  Null: every re-issue is compacted.
  float *xt1;
  SampleState *st1;
};

// tcgen05 contraction (xb_mvm_tc.cu).  fo == nullptr: split-K partial sums
// part[s][b][o] (split stride B x M; rows are x~ rows, n_dev = the number of
// valid rows when non-null); otherwise the cluster-fused output stage writes
// fo->Y (requires fo->o0 % 4 == 0 and splits <= 8).  bm_loop: run every BM
// re-issue inside the launch (returns false, and runs one pass, when the grid
// cannot be co-resident).
bool tc_gemm(Tile &t, bool transposed, bool x3, const float *Xt, int ldt, int B, float *part,
             int splits, const FusedOut *fo, const int *n_dev = nullptr, bool bm_loop = false);

} // namespace xb
