// xb_elem.cu -- fused elementwise passes over the tile storage (HBM-bound).
//
//   realize_kernel   d2d realization (proj/src/device.cpp:26-46), Philox normals
//   clip_kernel      set_weights clip to per-cell bounds (proj/src/tile.cpp:113-119)
//   temporal_kernel  decay / diffusion / reset (proj/src/tile.cpp:128-156)
//   program_kernel   PCM programming noise + drift exponents (proj/src/inference.cpp:34-61)
//   drift_kernel     w0 (t/t0)^-nu then clip (proj/src/inference.cpp:63-76)
//   nonfinite_kernel check_input's finiteness test on device-resident inputs
//                    (proj/src/tile.cpp:65-75)
//
// One thread per cell, row-major over [R][ld]; every random draw is addressed
// by the cell's GLOBAL (row, column) so row shards reproduce the whole tile.
#include <algorithm>

#include "xb_internal.h"

namespace xb {

namespace {

constexpr int EW_THREADS = 256;

inline dim3 ew_grid(int R, int C) { return dim3((C + 31) / 32, (R + 7) / 8); }

__device__ __forceinline__ bool ew_index(int R, int C, int &i, int &j) {
  j = blockIdx.x * 32 + (threadIdx.x & 31);
  i = blockIdx.y * 8 + (threadIdx.x >> 5);
  return i < R && j < C;
}

struct DevArgs {
  double dw_min, dw_min_dtod, up_down, up_down_dtod, w_max, w_min, w_max_dtod, w_min_dtod;
};

// proj/src/device.cpp:26-46: four Gaussians per cell (xi_dw, xi_ud, xi_max, xi_min)
__global__ void __launch_bounds__(EW_THREADS) realize_kernel(float2 *__restrict__ S,
                                                              float2 *__restrict__ Bd, int ld,
                                                              int R, int C, int row0,
                                                              DevArgs a, Key key) {
  int i, j;
  if (!ew_index(R, C, i, j)) return;
  float z0, z1, z2, z3;
  normal4((uint32_t)j, (uint32_t)(row0 + i), 0u, TAG_REALIZE << 24, key, z0, z1, z2, z3);
  const double fl = 0.01 * a.dw_min;
  const double dw = fmax(a.dw_min * (1.0 + a.dw_min_dtod * z0), fl);
  const double bias = a.up_down + a.up_down_dtod * z1;
  const size_t k = (size_t)i * ld + j;
  S[k] = make_float2((float)fmax(dw * (1.0 + bias), fl), (float)fmax(dw * (1.0 - bias), fl));
  Bd[k] = make_float2((float)fmax(a.w_max * (1.0 + a.w_max_dtod * z2), 0.01 * a.w_max),
                      (float)fmin(a.w_min * (1.0 + a.w_min_dtod * z3), 0.01 * a.w_min));
}

__global__ void __launch_bounds__(EW_THREADS) clip_kernel(float *__restrict__ W,
                                                           const float2 *__restrict__ Bd, int ld,
                                                           int R, int C) {
  int i, j;
  if (!ew_index(R, C, i, j)) return;
  const size_t k = (size_t)i * ld + j;
  const float2 p = Bd[k];
  W[k] = fminf(fmaxf(W[k], p.y), p.x);
}

__global__ void __launch_bounds__(EW_THREADS) temporal_xi_kernel(float *__restrict__ xi, int ld,
                                                                  int R, int C, int row0,
                                                                  Key key) {
  int i, j;
  if (!ew_index(R, C, i, j)) return;
  float z0, z1, z2, z3;
  normal4((uint32_t)j, (uint32_t)(row0 + i), 0u, TAG_TEMPORAL_XI << 24, key, z0, z1, z2, z3);
  const size_t k = (size_t)i * ld + j, plane = (size_t)R * ld;
  xi[k] = z0;
  xi[plane + k] = z1;
  xi[2 * plane + k] = z2;
}

struct TempArgs {
  double decay, decay_dtod, diff, diff_dtod, reset, reset_dtod;
};

// proj/src/tile.cpp:128-156
__global__ void __launch_bounds__(EW_THREADS) temporal_kernel(float *__restrict__ W,
                                                               const float2 *__restrict__ Bd,
                                                               const float *__restrict__ xi,
                                                               int ld, int R, int C, int row0,
                                                               TempArgs a, Key key,
                                                               uint32_t call) {
  int i, j;
  if (!ew_index(R, C, i, j)) return;
  const size_t k = (size_t)i * ld + j, plane = (size_t)R * ld;
  double w = W[k];
  uint32_t c0 = (uint32_t)j, c1 = (uint32_t)(row0 + i), c2 = call, c3 = TAG_TEMPORAL << 24;
  philox10(c0, c1, c2, c3, key);
  if (a.decay > 0.0) {
    const double r = fmin(fmax(a.decay * (1.0 + a.decay_dtod * xi[k]), 0.0), 1.0);
    w *= 1.0 - r;
  }
  if (a.diff > 0.0) {
    const double s = fmax(a.diff * (1.0 + a.diff_dtod * xi[plane + k]), 0.0);
    float z0, z1;
    box_muller(c0, c1, z0, z1);
    w += s * (double)z0;
  }
  if (a.reset > 0.0) {
    const double p = fmin(fmax(a.reset * (1.0 + a.reset_dtod * xi[2 * plane + k]), 0.0), 1.0);
    const bool hit = (p >= 1.0) || (p > 0.0 && (double)c2 * 2.3283064365386963e-10 < p);
    if (hit) w = 0.0;
  }
  const float2 pp = Bd[k];
  W[k] = fminf(fmaxf((float)w, pp.y), pp.x);
}

struct ProgArgs {
  double scale, c0, c1, c2, nu_mean, nu_std, nu_min, nu_max;
};

// The inference kernels stream 20-28 B per cell and are HBM-bound: each thread
// owns a quad of 4 consecutive cells of one row (16-B loads/stores; rows are
// 128-B aligned, ld a multiple of 32), a warp 128 columns.  Cells at j >= C
// (the row padding) are never touched.
inline unsigned ew4_blocks(int R, int ld) {
  const size_t quads = (size_t)R * (ld / 4);
  return (unsigned)((quads + EW_THREADS - 1) / EW_THREADS);
}

__device__ __forceinline__ bool ew4_index(int R, int C, int ld, int &i, int &j) {
  const size_t q = (size_t)blockIdx.x * EW_THREADS + threadIdx.x;
  const int qpr = ld >> 2;
  i = (int)(q / qpr);
  j = (int)(q - (size_t)i * qpr) * 4;
  return i < R && j < C;
}

// proj/src/inference.cpp:34-61: w = target + sigma(|target|) xi, clip -> w0;
// nu = clip(nu_mean (1 + nu_std xi'), nu_min, nu_max)
__device__ __forceinline__ void program_cell(float t32, float2 p, int j, int gi, const ProgArgs &a,
                                             Key key, float &w, float &nu) {
  float z0, z1, z2, z3;
  normal4((uint32_t)j, (uint32_t)gi, 0u, TAG_PROGRAM << 24, key, z0, z1, z2, z3);
  const double t = t32;
  const double at = fabs(t);
  const double sig = a.scale * (a.c0 + a.c1 * at + a.c2 * at * at);
  w = fminf(fmaxf((float)(t + sig * (double)z0), p.y), p.x);
  const double v = a.nu_mean * (1.0 + a.nu_std * (double)z1);
  nu = (float)fmin(fmax(v, a.nu_min), a.nu_max);
}

__global__ void __launch_bounds__(EW_THREADS) program_kernel(
    float *__restrict__ W, float *__restrict__ w0, float *__restrict__ nu,
    const float2 *__restrict__ Bd, const float *__restrict__ target, int ld, int R, int C,
    int row0, ProgArgs a, Key key) {
  int i, j;
  if (!ew4_index(R, C, ld, i, j)) return;
  const size_t k = (size_t)i * ld + j;
  const float *tr = target + (size_t)i * C + j;
  if (j + 4 <= C) {
    float tv[4];
    if ((C & 3) == 0) {
      const float4 t4 = __ldcs(reinterpret_cast<const float4 *>(tr));
      tv[0] = t4.x, tv[1] = t4.y, tv[2] = t4.z, tv[3] = t4.w;
    } else {
      for (int e = 0; e < 4; ++e) tv[e] = __ldcs(tr + e);
    }
    const float4 b01 = __ldcs(reinterpret_cast<const float4 *>(Bd + k));
    const float4 b23 = __ldcs(reinterpret_cast<const float4 *>(Bd + k + 2));
    const float2 pb[4] = {{b01.x, b01.y}, {b01.z, b01.w}, {b23.x, b23.y}, {b23.z, b23.w}};
    float w[4], n[4];
    for (int e = 0; e < 4; ++e) program_cell(tv[e], pb[e], j + e, row0 + i, a, key, w[e], n[e]);
    const float4 w4 = make_float4(w[0], w[1], w[2], w[3]);
    __stcs(reinterpret_cast<float4 *>(W + k), w4);
    __stcs(reinterpret_cast<float4 *>(w0 + k), w4);
    __stcs(reinterpret_cast<float4 *>(nu + k), make_float4(n[0], n[1], n[2], n[3]));
  } else {
    for (int e = 0; j + e < C; ++e) {
      float w, n;
      program_cell(tr[e], Bd[k + e], j + e, row0 + i, a, key, w, n);
      W[k + e] = w;
      w0[k + e] = w;
      nu[k + e] = n;
    }
  }
}

// proj/src/inference.cpp:63-76 with log2(t/t0) precomputed in fp64 on the host
__device__ __forceinline__ float drift_cell(float w0, float nu, float2 p, double log2_ratio) {
  const double f = exp2(-(double)nu * log2_ratio);
  return fminf(fmaxf((float)((double)w0 * f), p.y), p.x);
}

__global__ void __launch_bounds__(EW_THREADS) drift_kernel(float *__restrict__ W,
                                                            const float *__restrict__ w0,
                                                            const float *__restrict__ nu,
                                                            const float2 *__restrict__ Bd, int ld,
                                                            int R, int C, double log2_ratio) {
  int i, j;
  if (!ew4_index(R, C, ld, i, j)) return;
  const size_t k = (size_t)i * ld + j;
  if (j + 4 <= C) {
    const float4 a = __ldcs(reinterpret_cast<const float4 *>(w0 + k));
    const float4 n = __ldcs(reinterpret_cast<const float4 *>(nu + k));
    const float4 b01 = __ldcs(reinterpret_cast<const float4 *>(Bd + k));
    const float4 b23 = __ldcs(reinterpret_cast<const float4 *>(Bd + k + 2));
    float4 o;
    o.x = drift_cell(a.x, n.x, make_float2(b01.x, b01.y), log2_ratio);
    o.y = drift_cell(a.y, n.y, make_float2(b01.z, b01.w), log2_ratio);
    o.z = drift_cell(a.z, n.z, make_float2(b23.x, b23.y), log2_ratio);
    o.w = drift_cell(a.w, n.w, make_float2(b23.z, b23.w), log2_ratio);
    __stcs(reinterpret_cast<float4 *>(W + k), o);
  } else {
    for (int e = 0; j + e < C; ++e) W[k + e] = drift_cell(w0[k + e], nu[k + e], Bd[k + e], log2_ratio);
  }
}

// ORs `bit` into *flag if any of v[0..n) is Inf or NaN (exponent all ones):
// a streaming read, 16-B loads when the pointer allows them
__global__ void __launch_bounds__(EW_THREADS) nonfinite_kernel(const float *__restrict__ v,
                                                               size_t n, int bit, int *flag) {
  const size_t tid = (size_t)blockIdx.x * EW_THREADS + threadIdx.x;
  const size_t nth = (size_t)gridDim.x * EW_THREADS;
  uint32_t bad = 0;
  size_t head = 0;
  if (((uintptr_t)v & 15) == 0) {
    const uint4 *v4 = reinterpret_cast<const uint4 *>(v);
    const size_t n4 = n / 4;
    for (size_t k = tid; k < n4; k += nth) {
      const uint4 q = __ldcs(v4 + k);
      bad |= (~q.x & 0x7f800000u) == 0 || (~q.y & 0x7f800000u) == 0 ||
             (~q.z & 0x7f800000u) == 0 || (~q.w & 0x7f800000u) == 0;
    }
    head = n4 * 4;
  }
  const uint32_t *u = reinterpret_cast<const uint32_t *>(v);
  for (size_t k = head + tid; k < n; k += nth) bad |= (~__ldcs(u + k) & 0x7f800000u) == 0;
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, bit);
}

struct EffArgs {
  const float *w[XB_MAX_CELL_DEVICES];
  double g[XB_MAX_CELL_DEVICES];
  int K;
};

// proj/src/compound.cpp:66-80: effective weight of a unit cell, members in order
__global__ void __launch_bounds__(EW_THREADS) effective_kernel(float *__restrict__ weff,
                                                               EffArgs a, int ld, int R, int C) {
  int i, j;
  if (!ew_index(R, C, i, j)) return;
  const size_t k = (size_t)i * ld + j;
  double acc = 0.0;
  for (int m = 0; m < a.K; ++m) acc += a.g[m] * (double)a.w[m][k];
  weff[k] = (float)acc;
}

} // namespace

void launch_effective(float *weff, const float *const *w, const double *g, int K, int R, int C,
                      int ld, cudaStream_t s) {
  if (R == 0 || K < 1 || K > XB_MAX_CELL_DEVICES) return;
  EffArgs a;
  a.K = K;
  for (int m = 0; m < K; ++m) {
    a.w[m] = w[m];
    a.g[m] = g[m];
  }
  effective_kernel<<<ew_grid(R, C), EW_THREADS, 0, s>>>(weff, a, ld, R, C);
  count_launch();
  XB_CUDA(cudaGetLastError());
}

__global__ void empty_kernel() {}

void launch_empty(cudaStream_t s) {
  empty_kernel<<<1, 32, 0, s>>>();
  XB_CUDA(cudaGetLastError());
}

void launch_nonfinite(const float *v, size_t n, int bit, int *flag, cudaStream_t s) {
  if (n == 0) return;
  const size_t blocks = std::min<size_t>((n / 4 + EW_THREADS - 1) / EW_THREADS + 1, 148 * 8);
  nonfinite_kernel<<<(unsigned)blocks, EW_THREADS, 0, s>>>(v, n, bit, flag);
  count_launch();
  XB_CUDA(cudaGetLastError());
}

void launch_realize(Tile &t) {
  if (t.R == 0) return;
  const xb_device_params &d = t.cfg.device;
  DevArgs a{d.dw_min, d.dw_min_dtod, d.up_down, d.up_down_dtod, d.w_max, d.w_min, d.w_max_dtod,
            d.w_min_dtod};
  realize_kernel<<<ew_grid(t.R, t.C), EW_THREADS, 0, t.stream>>>(t.steps(), t.bounds(), t.ld, t.R, t.C, t.row0, a,
                                                                  t.k_realize);
  count_launch();
  XB_CUDA(cudaGetLastError());
}

void launch_clip(Tile &t) {
  if (t.R == 0) return;
  clip_kernel<<<ew_grid(t.R, t.C), EW_THREADS, 0, t.stream>>>(t.W, t.bounds(), t.ld, t.R, t.C);
  count_launch();
  XB_CUDA(cudaGetLastError());
}

void launch_temporal_xi(Tile &t) {
  if (t.R == 0) return;
  temporal_xi_kernel<<<ew_grid(t.R, t.C), EW_THREADS, 0, t.stream>>>(t.xi, t.ld, t.R, t.C,
                                                                      t.row0, t.k_tinit);
  count_launch();
  XB_CUDA(cudaGetLastError());
}

void launch_temporal(Tile &t, const xb_temporal_params &tp, uint32_t call) {
  if (t.R == 0) return;
  TempArgs a{tp.decay_rate, tp.decay_dtod, tp.diffusion_sigma, tp.diffusion_dtod, tp.reset_prob,
             tp.reset_dtod};
  temporal_kernel<<<ew_grid(t.R, t.C), EW_THREADS, 0, t.stream>>>(
      t.W, t.bounds(), t.xi, t.ld, t.R, t.C, t.row0, a, t.k_temporal, call);
  count_launch();
  XB_CUDA(cudaGetLastError());
}

void launch_program(Tile &t, const float *target_dev, const xb_inference_model &m, Key key) {
  if (t.R == 0) return;
  ProgArgs a{m.prog_noise_scale, m.prog_c0, m.prog_c1, m.prog_c2,
             m.nu_mean,          m.nu_std,  m.nu_min,  m.nu_max};
  program_kernel<<<ew4_blocks(t.R, t.ld), EW_THREADS, 0, t.stream>>>(
      t.W, t.w0, t.nu, t.bounds(), target_dev, t.ld, t.R, t.C, t.row0, a, key);
  count_launch();
  XB_CUDA(cudaGetLastError());
}

void launch_drift(Tile &t, double ratio) {
  if (t.R == 0) return;
  drift_kernel<<<ew4_blocks(t.R, t.ld), EW_THREADS, 0, t.stream>>>(t.W, t.w0, t.nu, t.bounds(), t.ld, t.R,
                                                                t.C, log2(ratio));
  count_launch();
  XB_CUDA(cudaGetLastError());
}

} // namespace xb
