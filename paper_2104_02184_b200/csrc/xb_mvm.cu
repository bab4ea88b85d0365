// xb_mvm.cu -- the noisy analog MVM (paper Eq. 1), proj/src/io.cpp:93-149.
//
// For B samples at once (the weights are stationary across the batch):
//   prep_kernel      per sample: alpha = max|x| (abs_max), x~ = Q_dac(x / (alpha 2^m))
//                    + sigma_inp xi (fp64 converter arithmetic, like the
//                    reference); ||x~||^2 for the weight-noise fold
//   mvm_*_kernel     acc[b][o] = sum_k W x~ (fp32 FMA SIMT path; the tcgen05
//                    path lives in xb_mvm_tc.cu)
//   epilogue_kernel  v = acc + sigma_w ||x~|| zeta + sigma_out xi;
//                    y = alpha 2^m Q_adc(v); zero-input samples get Q_adc(sigma_out xi)
//                    (io.cpp:107-115).  Under bound management a sample whose
//                    |v| reaches output_bound is re-issued with m + 1.
//
// Weight noise: sum_j (w_ij + sigma_w xi_ij) x~_j = sum_j w_ij x~_j + sigma_w
// ||x~|| zeta_i exactly in distribution (independent xi_ij), so the per-use
// d_out x d_in Gaussian draws of the reference become one normal per output.
#include <cstdlib>

#include "xb_mvm_common.cuh"

namespace xb {

namespace {

constexpr int PREP_THREADS = 512;
constexpr int PREP_VPT = 8; // values per thread kept in registers (n <= 4096)

__device__ __forceinline__ float block_max(float m, float *red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  m = warp_max(m);
  if (lane == 0) red[warp] = m;
  __syncthreads();
  if (warp == 0) {
    m = lane < nw ? red[lane] : 0.f;
    m = warp_max(m);
    if (lane == 0) red[32] = m;
  }
  __syncthreads();
  return red[32];
}

__global__ void __launch_bounds__(PREP_THREADS) prep_kernel(const float *__restrict__ X, int n,
                                                             int ldx, float *__restrict__ Xt,
                                                             int ldt,
                                                             SampleState *__restrict__ st,
                                                             IoDev io, Key key, uint64_t seq0,
                                                             int first_pass,
                                                             const float *__restrict__ amax_in,
                                                             int *__restrict__ sat,
                                                             const int *__restrict__ map,
                                                             int in0) {
  // in0: global index of input 0 (row-shard backward: the shard's first row),
  // so the input-noise counters match the unsharded tile's
  // map != nullptr: a compacted bound-management re-issue -- block i prepares
  // sample map[i] into x~ row i (compact_kernel already re-armed the flags)
  const int b = map ? map[blockIdx.x] : blockIdx.x;
  SampleState s = st[b];
  if (map) {
    s.m += 1;
  } else if (!first_pass) { // bound management: re-issue the samples that saturated
    const int again = s.active && sat[b];
    __syncthreads(); // every thread has read the flag before it is re-armed
    if (threadIdx.x == 0) sat[b] = 0;
    if (!again) {
      if (threadIdx.x == 0 && s.active) {
        s.active = 0;
        st[b] = s;
      }
      return;
    }
    s.m += 1;
  }
  const float *x = X + (size_t)b * ldx;
  float *xt = Xt + (size_t)blockIdx.x * ldt;
  __shared__ float red[33];
  // the sample stays in registers between the max and the conversion when it fits
  const bool in_regs = n <= PREP_THREADS * PREP_VPT;
  float v[PREP_VPT];
  if (in_regs) {
#pragma unroll
    for (int u = 0; u < PREP_VPT; ++u) {
      const int j = threadIdx.x + u * PREP_THREADS;
      v[u] = j < n ? x[j] : 0.f;
    }
  }
  if (first_pass) {
    float m = 0.f;
    if (amax_in) {
      m = amax_in[b];
    } else {
      if (in_regs) {
#pragma unroll
        for (int u = 0; u < PREP_VPT; ++u) m = fmaxf(m, fabsf(v[u]));
      } else {
        for (int j = threadIdx.x; j < n; j += blockDim.x) m = fmaxf(m, fabsf(x[j]));
      }
      m = block_max(m, red);
    }
    s.alpha = (m == 0.f) ? 0.f : (io.nm_absmax ? m : 1.f);
    s.m = 0;
    s.active = 1;
  }
  const uint64_t seq = seq0 + (uint64_t)b;
  const double inv = (s.alpha == 0.f) ? 0.0 : 1.0 / ((double)s.alpha * pow2i(s.m));
  auto convert = [&](float xv, int j) -> float {
    if (io.perfect) return xv;
    if (s.alpha == 0.f) return 0.f;
    double q = quantize((double)xv * inv, io.dac); // x / alpha, then the DAC (io.cpp:122-130)
    if (io.sigma_inp > 0.0) {
      const float z = normal1((uint32_t)(j + in0), (uint32_t)seq, (uint32_t)(seq >> 32) | (s.m << 24),
                              TAG_IN_NOISE << 24, key);
      q += io.sigma_inp * (double)z;
    }
    return (float)q;
  };
  float nrm = 0.f;
  if (in_regs) {
#pragma unroll
    for (int u = 0; u < PREP_VPT; ++u) {
      const int j = threadIdx.x + u * PREP_THREADS;
      if (j < n) {
        const float f = convert(v[u], j);
        xt[j] = f;
        nrm = fmaf(f, f, nrm);
      }
    }
  } else {
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const float f = convert(x[j], j);
      xt[j] = f;
      nrm = fmaf(f, f, nrm);
    }
  }
  nrm = warp_sum(nrm);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = nrm;
  __syncthreads();
  if (threadIdx.x == 0) {
    float tot = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
    s.norm = sqrtf(tot);
    st[b] = s;
  }
}

// Bound-management bookkeeping between passes: samples that saturated in the
// last pass (and are still active) are listed in map[0..n) -- in any order:
// each sample's column of the contraction is independent of its position --
// the others are retired; all flags are re-armed for the next pass.
__global__ void __launch_bounds__(256) compact_kernel(int *__restrict__ sat,
                                                      SampleState *__restrict__ st, int B,
                                                      int *__restrict__ map,
                                                      int *__restrict__ count) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  bool again = false;
  if (b < B) {
    SampleState s = st[b];
    again = s.active && sat[b];
    sat[b] = 0;
    if (!again && s.active) {
      s.active = 0;
      st[b] = s;
    }
  }
  const unsigned m = __ballot_sync(0xffffffffu, again);
  int base = 0;
  if ((threadIdx.x & 31) == 0 && m) base = atomicAdd(count, __popc(m));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (again) map[base + __popc(m & ((1u << (threadIdx.x & 31)) - 1u))] = b;
}

// --------------------------------------------------------------- SIMT GEMM
// acc[b][o] = sum_k A(o, k) x~[b][k];  forward: A(o,k) = W[o][k] (K-major),
// backward: A(o,k) = W[k][o] (M-major).  Tile 64 (o) x 64 (b) x 16 (k),
// 256 threads x (4 x 4) outputs.  Samples of inactive BM passes are skipped
// per tile.
template <bool TRANS>
__global__ void __launch_bounds__(256) mvm_simt_kernel(const float *__restrict__ W, int ldw,
                                                        int M, int K, const float *__restrict__ Xt,
                                                        int ldt, int B, float *__restrict__ acc,
                                                        int lda, const SampleState *__restrict__ st,
                                                        int first_pass) {
  __shared__ float As[16][64 + 4];
  __shared__ float Bs[16][64 + 4];
  __shared__ int any_active;
  const int m0 = blockIdx.x * 64, b0 = blockIdx.y * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  if (!first_pass) {
    if (threadIdx.x == 0) any_active = 0;
    __syncthreads();
    if (threadIdx.x < 64 && b0 + threadIdx.x < B && st[b0 + threadIdx.x].active) any_active = 1;
    __syncthreads();
    if (!any_active) return;
  }
  float c[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    // A tile
    for (int t = threadIdx.x; t < 64 * 16; t += 256) {
      int kk, mm;
      float v = 0.f;
      if (TRANS) {
        kk = t >> 6;
        mm = t & 63;
        if (k0 + kk < K && m0 + mm < M) v = W[(size_t)(k0 + kk) * ldw + m0 + mm];
      } else {
        mm = t >> 4;
        kk = t & 15;
        if (k0 + kk < K && m0 + mm < M) v = W[(size_t)(m0 + mm) * ldw + k0 + kk];
      }
      As[kk][mm] = v;
    }
    for (int t = threadIdx.x; t < 64 * 16; t += 256) {
      const int nn = t >> 4, kk = t & 15;
      float v = 0.f;
      if (k0 + kk < K && b0 + nn < B) v = Xt[(size_t)(b0 + nn) * ldt + k0 + kk];
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], bb[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) a[r] = As[kk][ty * 4 + r];
#pragma unroll
      for (int q = 0; q < 4; ++q) bb[q] = Bs[kk][tx * 4 + q];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q) c[r][q] = fmaf(a[r], bb[q], c[r][q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int b = b0 + tx * 4 + q;
    if (b >= B) continue;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int o = m0 + ty * 4 + r;
      if (o < M) acc[(size_t)b * lda + o] = c[r][q];
    }
  }
}

// --------------------------------------------------------------- epilogue
// one thread = one group of 4 outputs of one sample (xb_mvm_common.cuh)
__global__ void __launch_bounds__(256) epilogue_kernel(const float *__restrict__ acc, int lda,
                                                        int nsplit, size_t split_stride, int M,
                                                        int o0, float *__restrict__ Y, int ldy,
                                                        SampleState *__restrict__ st, IoDev io,
                                                        Key key, uint64_t seq0,
                                                        int *__restrict__ sat, int first_pass,
                                                        int B, int pass_slot,
                                                        const int *__restrict__ map) {
  // acc row blockIdx.y holds sample b (compacted re-issue: b = map[row])
  const int row = blockIdx.y, b = map ? map[row] : row;
  const SampleState s = st[b];
  if (!first_pass && !s.active) return;
  const int g = (o0 >> 2) + blockIdx.x * blockDim.x + threadIdx.x;
  if (4 * g >= o0 + M) return;
  float a[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int o = 4 * g + k - o0;
    if (o < 0 || o >= M) continue;
    a[k] = acc[(size_t)row * lda + o];
    for (int sp = 1; sp < nsplit; ++sp) a[k] += acc[sp * split_stride + (size_t)row * lda + o];
  }
  const bool hit = epilogue_group4(a, g, o0, M, s, io, key, seq0 + (uint64_t)b,
                                   Y + (size_t)b * ldy);
  bm_flag(hit, s, io, sat, b, B, pass_slot);
}

// Row-shard backward, phase 1: the shard's column sums plus its share of the
// weight-noise fold (independent per shard: the variances of the shards add
// up to sigma_w^2 ||d~||^2 over all rows).  No output noise, ADC or alpha yet.
__global__ void __launch_bounds__(256) partial_kernel(const float *__restrict__ acc, int M,
                                                       int nsplit, size_t split_stride,
                                                       float *__restrict__ P,
                                                       const SampleState *__restrict__ st,
                                                       IoDev io, Key key, uint64_t seq0,
                                                       uint32_t shard_tag) {
  const int b = blockIdx.y;
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= M) return;
  const SampleState s = st[b];
  float v = acc[(size_t)b * M + o];
  for (int sp = 1; sp < nsplit; ++sp) v += acc[sp * split_stride + (size_t)b * M + o];
  if (!io.perfect && io.sigma_w > 0.0 && s.alpha != 0.f) {
    const uint64_t seq = seq0 + (uint64_t)b;
    const float z = normal1((uint32_t)o, (uint32_t)seq, (uint32_t)(seq >> 32), shard_tag, key);
    v += (float)(io.sigma_w * (double)s.norm * (double)z);
  }
  P[(size_t)b * M + o] = v;
}

// Row-shard backward, phase 2 (after the sum over shards): output noise, ADC
// and alpha act on the reduced column sums, as in proj/src/io.cpp:143-146.
// Same noise groups as epilogue_kernel (o0 = 0, m = 0), so the split-phase
// backward reproduces the whole-tile backward bit for bit.
__global__ void __launch_bounds__(256) finish_kernel(const float *__restrict__ Psum, int M,
                                                      const float *__restrict__ amax,
                                                      float *__restrict__ Y, IoDev io, Key key,
                                                      uint64_t seq0) {
  const int b = blockIdx.y;
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (4 * g >= M) return;
  const float m = amax[b];
  SampleState s;
  s.alpha = (m == 0.f) ? 0.f : (io.nm_absmax ? m : 1.f);
  s.norm = 0.f;
  s.m = 0;
  s.active = 1;
  float a[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (4 * g + k < M) a[k] = Psum[(size_t)b * M + 4 * g + k];
  // the weight-noise fold is already in the partial sums (partial_kernel):
  // only the output noise, the ADC and alpha act here, with the same noise
  // words and arithmetic as the whole-tile output stage
  io.sigma_w = 0.0;
  epilogue_group4(a, g, 0, M, s, io, key, seq0 + (uint64_t)b, Y + (size_t)b * M);
}

struct MvmScratch {
  float *xt;
  float *acc;
  SampleState *st;
  int *sat; // [B] flags, then one saturation counter per BM pass, then the compaction counters
  int *map; // [B] compacted re-issue list
};

MvmScratch carve(Tile &t, int B, int K, int M, int nsplit) {
  const size_t xt_b = (size_t)B * K * sizeof(float);
  const size_t acc_b = (size_t)nsplit * B * M * sizeof(float);
  const size_t st_b = (size_t)B * sizeof(SampleState);
  const size_t sat_b = (size_t)(B + 64) * sizeof(int); // flags + per-pass counters
  const size_t map_b = (size_t)B * sizeof(int);
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  char *p = (char *)t.s_io.get(al(xt_b) + al(acc_b) + al(st_b) + al(sat_b) + al(map_b));
  MvmScratch s;
  s.xt = (float *)p;
  s.acc = (float *)(p + al(xt_b));
  s.st = (SampleState *)(p + al(xt_b) + al(acc_b));
  s.sat = (int *)(p + al(xt_b) + al(acc_b) + al(st_b));
  s.map = (int *)(p + al(xt_b) + al(acc_b) + al(st_b) + al(sat_b));
  return s;
}

template <bool TRANS>
void gemm(Tile &t, const MvmScratch &s, int M, int K, int ldt, int B, int first) {
  dim3 grid((M + 63) / 64, (B + 63) / 64);
  mvm_simt_kernel<TRANS><<<grid, 256, 0, t.stream>>>(t.W, t.ld, M, K, s.xt, ldt, B, s.acc, M,
                                                     s.st, first);
  count_launch();
  XB_CUDA(cudaGetLastError());
}

// XB_MVM_UNFUSED=1 forces the split-K partials + epilogue kernel path: the
// parity tests run both and require bit-identical outputs
static bool unfused_requested() {
  const char *e = getenv("XB_MVM_UNFUSED");
  return e && e[0] == '1';
}

// one full noisy MVM in direction TRANS (forward: false)
// tensor-core contraction at TF32 / 3xTF32 (B >= 16); the fp32 SIMT kernel
// otherwise (exact-fp32 parity mode, tiny batches)
static bool use_tc(const Tile &t, int B) {
  return (t.cfg.mvm_precision == XB_MVM_TF32 || t.cfg.mvm_precision == XB_MVM_TF32X3) && B >= 16;
}

template <bool TRANS>
void run_mvm(Tile &t, const float *dIn, int B, float *dOut, const IoDev &io_in, Key key,
             uint64_t seq0, const float *amax_in, bool skip_epilogue, float *dPartial) {
  const int K = TRANS ? t.R : t.C; // contraction length
  const int M = TRANS ? t.C : t.R; // outputs
  if (B <= 0) return;
  const bool x3 = t.cfg.mvm_precision == XB_MVM_TF32X3;
  const bool tc = use_tc(t, B);
  IoDev io = io_in;
  io.exact = !tc; // fp64 output stage only behind the exact fp32 contraction
  const int o0 = TRANS ? 0 : t.row0; // global index of output 0 (noise counters)
  // the output stage runs inside the tcgen05 kernel (K-splits reduced over a
  // thread-block cluster) unless the caller wants raw partial sums, the noise
  // groups of 4 outputs do not align with the tile, or a cluster would exceed
  // the portable 8 CTAs
  // (both paths use the same K-splits, so they agree bit for bit)
  const int splits = tc ? tc_used_splits(K, std::min(8, tc_splits(M, K, x3))) : 1;
  const bool fused = tc && !skip_epilogue && (o0 & 3) == 0 && !unfused_requested();
  const int ldt = (K + 3) & ~3; // x~ rows padded to 16 bytes (TMA global stride)
  MvmScratch s = carve(t, B, ldt, M, fused ? 0 : splits);
  if (io.bm) XB_CUDA(cudaMemsetAsync(s.sat, 0, sizeof(int) * (B + 64), t.stream));
  const int passes = io.bm ? 1 + io.bm_max_iter : 1;
  int nrun = B;             // samples (rows of x~) in this pass
  const int *map = nullptr; // tensor-core re-issues: the compacted list of saturated samples
  for (int pass = 0; pass < passes; ++pass) {
    const int first = pass == 0;
    prep_kernel<<<nrun, PREP_THREADS, 0, t.stream>>>(dIn, K, K, s.xt, ldt, s.st, io, key, seq0,
                                                      first, amax_in, s.sat, map,
                                                      TRANS ? t.row0 : 0);
    count_launch();
    XB_CUDA(cudaGetLastError());
    int nsplit = 1;
    if (fused) {
      FusedOut fo{dOut, M, s.st, io, key, seq0, s.sat, first, B, pass, o0, 0, map};
      tc_gemm(t, TRANS, x3, s.xt, ldt, nrun, nullptr, splits, &fo);
    } else if (tc) {
      tc_gemm(t, TRANS, x3, s.xt, ldt, nrun, s.acc, splits, nullptr);
      nsplit = splits;
    } else { // SIMT: re-issues run over the whole batch, skipping inactive tiles
      gemm<TRANS>(t, s, M, K, ldt, B, first);
    }
    if (skip_epilogue) { // row shard: partial sums + this shard's weight-noise fold
      dim3 eg((M + 255) / 256, B);
      partial_kernel<<<eg, 256, 0, t.stream>>>(s.acc, M, nsplit, (size_t)B * M, dPartial, s.st,
                                               io, key, seq0,
                                               (TAG_W_NOISE << 24) | (uint32_t)t.row0);
      count_launch();
      XB_CUDA(cudaGetLastError());
      return;
    }
    if (!fused) {
      dim3 eg((out_groups(o0, M) + 255) / 256, nrun);
      epilogue_kernel<<<eg, 256, 0, t.stream>>>(s.acc, M, nsplit, (size_t)nrun * M, M, o0, dOut,
                                                M, s.st, io, key, seq0, s.sat, first, B, pass,
                                                map);
      count_launch();
      XB_CUDA(cudaGetLastError());
    }
    if (io.bm && pass + 1 < passes) {
      // bound management: re-issue while some sample saturated.  The epilogue
      // counted them; the count crosses to the host (one 4-byte read and a
      // stream sync per pass with BM on).  On the tensor cores only the
      // saturated samples are recomputed: compact_kernel lists them, retires
      // the rest and re-arms the flags (the SIMT path's prep does the latter).
      if (!t.bm_count) XB_CUDA(cudaMallocHost(&t.bm_count, sizeof(int)));
      XB_CUDA(cudaMemcpyAsync(t.bm_count, s.sat + B + pass, sizeof(int),
                              cudaMemcpyDeviceToHost, t.stream));
      XB_CUDA(cudaStreamSynchronize(t.stream));
      const int nsat = *t.bm_count;
      if (nsat == 0) break;
      if (tc) {
        compact_kernel<<<(B + 255) / 256, 256, 0, t.stream>>>(s.sat, s.st, B, s.map,
                                                              s.sat + B + 32 + pass);
        count_launch();
        XB_CUDA(cudaGetLastError());
        map = s.map;
        nrun = nsat;
      }
    }
  }
}

} // namespace

IoDev make_io(const xb_io_params &io) {
  IoDev d;
  d.dac = make_quant(io.input_bound, io.dac_bits);
  d.adc = make_quant(io.output_bound, io.adc_bits);
  d.sigma_inp = io.sigma_inp;
  d.sigma_out = io.sigma_out;
  d.sigma_w = io.sigma_w;
  d.nm_absmax = io.noise_management == XB_NM_ABS_MAX;
  d.perfect = io.is_perfect;
  d.bm = io.bound_management == XB_BM_ITERATIVE && !io.is_perfect;
  d.bm_max_iter = io.bm_max_iter;
  d.exact = 1;
  return d;
}

void mvm_forward(Tile &t, const float *dX, int B, float *dY, const IoDev &io, Key key,
                 uint64_t seq0) {
  run_mvm<false>(t, dX, B, dY, io, key, seq0, nullptr, false, nullptr);
}

void mvm_backward(Tile &t, const float *dD, int B, float *dG, const IoDev &io, Key key,
                  uint64_t seq0, const float *amax_global, bool partial_only, float *dP) {
  run_mvm<true>(t, dD, B, dG, io, key, seq0, amax_global, partial_only, dP);
}

void mvm_backward_finish(Tile &t, const float *dPsum, int B, const float *amax_global, float *dG,
                         const IoDev &io, Key key, uint64_t seq0) {
  if (B <= 0) return;
  if (!amax_global) raise("backward_finish: the global max|d| per sample is required");
  IoDev io2 = io;
  io2.exact = !use_tc(t, B);
  dim3 eg((out_groups(0, t.C) + 255) / 256, B);
  finish_kernel<<<eg, 256, 0, t.stream>>>(dPsum, t.C, amax_global, dG, io2, key, seq0);
  count_launch();
  XB_CUDA(cudaGetLastError());
}

} // namespace xb
