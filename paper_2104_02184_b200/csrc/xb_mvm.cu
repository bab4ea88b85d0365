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
#include <algorithm>
#include <cstdlib>

#include "xb_mvm_common.cuh"

#ifdef XB_TC_TRACE
// experiment builds only: globaltimer at the start and end of every prep block
__device__ unsigned long long g_prep_trace[4096][4];
extern "C" __attribute__((visibility("default"))) int xb_debug_prep_trace(unsigned long long *out,
                                                                            int n) {
  return (int)cudaMemcpyFromSymbol(out, g_prep_trace,
                                   sizeof(unsigned long long) * 4 * (size_t)(n < 4096 ? n : 4096));
}
__device__ __forceinline__ void prep_stamp(int k) {
  unsigned long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  if (threadIdx.x == 0 && blockIdx.x < 4096) g_prep_trace[blockIdx.x][k] = v;
}
#else
__device__ __forceinline__ void prep_stamp(int) {}
#endif

namespace xb {

namespace {

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

constexpr int PREP_THREADS = XB_PREP_THREADS;

// Pass 0: alpha = max|x| per sample (abs-max; or the all-reduced global value
// of a row shard), x~ at m = 0, ||x~||.  Block 0 also clears the
// bound-management buffers of the call (flags, counters, grid barriers), so
// no memset precedes the contraction.
__global__ void __launch_bounds__(PREP_THREADS) prep_kernel(
    const float *__restrict__ X, int n, float *__restrict__ Xt, int ldt,
    SampleState *__restrict__ st, IoDev io, Key key, uint64_t seq0,
    const float *__restrict__ amax_in, int in0, int *__restrict__ bm_clear, int bm_words) {
  // the contraction (a programmatic dependent) may start its prologue and
  // W loads now; it waits for this grid before touching x~ / st / flags
  asm volatile("griddepcontrol.launch_dependents;");
  prep_stamp(0);
  const int b = blockIdx.x;
  __shared__ float red[33];
  if (bm_clear && b == 0)
    for (int i = threadIdx.x; i < bm_words; i += blockDim.x) bm_clear[i] = 0;
  const float *x = X + (size_t)b * n;
  // short rows (the usual case): one read of x into registers serves the
  // abs-max and the DAC
  const bool regs = n <= (int)blockDim.x * PREP_VPT;
  float v[PREP_VPT];
  float m = 0.f;
  if (regs) {
#pragma unroll
    for (int u = 0; u < PREP_VPT; ++u) {
      const int j = threadIdx.x + u * (int)blockDim.x;
      v[u] = j < n ? __ldcs(x + j) : 0.f;
      m = fmaxf(m, fabsf(v[u]));
    }
  } else if (!amax_in) {
    for (int j = threadIdx.x; j < n; j += blockDim.x) m = fmaxf(m, fabsf(x[j]));
  }
  prep_stamp(2);
  if (amax_in)
    m = amax_in[b];
  else
    m = block_max(m, red);
  prep_stamp(3);
  SampleState s;
  s.alpha = (m == 0.f) ? 0.f : (io.nm_absmax ? m : 1.f);
  s.m = 0;
  s.active = 1;
  const uint64_t seq = seq0 + (uint64_t)b;
  s.norm = regs ? prep_row_vals(v, n, Xt + (size_t)b * ldt, s, io, key, seq, in0, red)
                : prep_row(x, n, Xt + (size_t)b * ldt, s, io, key, seq, in0, red);
  if (threadIdx.x == 0) st[b] = s;
  prep_stamp(1);
}

// Re-issue prep (host-driven passes): block c < *count prepares the x~ row c
// of sample map[c] at m + 1.
__global__ void __launch_bounds__(PREP_THREADS) reprep_kernel(
    const float *__restrict__ X, int n, float *__restrict__ Xt, int ldt,
    SampleState *__restrict__ st, IoDev io, Key key, uint64_t seq0, int in0,
    const int *__restrict__ map, const int *__restrict__ count) {
  const int c = blockIdx.x;
  if (c >= *count) return;
  __shared__ float red[33];
  const int b = map[c];
  SampleState s = st[b];
  s.m += 1;
  s.norm = prep_row(X + (size_t)b * n, n, Xt + (size_t)c * ldt, s, io, key, seq0 + (uint64_t)b,
                    in0, red);
  if (threadIdx.x == 0) st[b] = s;
}

// Host-driven re-issue bookkeeping (one block per N slab): the samples whose
// pass-(p-1) flag is set, ascending, into map; their number into *count; the
// flags pass p will write are cleared.
__global__ void __launch_bounds__(256) compact_kernel(int *__restrict__ flags, int nb, int n0,
                                                      int prev_pass, int *__restrict__ map,
                                                      int *__restrict__ count) {
  __shared__ int cnt[40];
  const int n = block_compact(flags + (prev_pass & 1) * nb, nb, n0, map, cnt);
  int *nf = flags + ((prev_pass + 1) & 1) * nb;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) nf[i] = 0;
  if (threadIdx.x == 0) *count = n;
}

// --------------------------------------------------------------- SIMT GEMM
// acc[b][o] = sum_k A(o, k) x~[b][k];  forward: A(o,k) = W[o][k] (K-major),
// backward: A(o,k) = W[k][o] (M-major).  Tile 64 (o) x 64 (b) x 16 (k),
// 256 threads x (4 x 4) outputs.  n_rows != nullptr: a compacted BM
// re-issue, only the first *n_rows rows of x~ are valid.
template <bool TRANS>
__global__ void __launch_bounds__(256) mvm_simt_kernel(const float *__restrict__ W, int ldw,
                                                        int M, int K, const float *__restrict__ Xt,
                                                        int ldt, int B, float *__restrict__ acc,
                                                        int lda, const int *__restrict__ n_rows) {
  __shared__ float As[16][64 + 4];
  __shared__ float Bs[16][64 + 4];
  const int m0 = blockIdx.x * 64, b0 = blockIdx.y * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  if (n_rows) B = min(B, *n_rows);
  if (b0 >= B) return;
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

// --------------------------------------------------------------- GEMV
// Small batches (B <= 15: every per-sample call of the reference API) stream
// W once at HBM rate with every sample's accumulator in registers (the 64 x
// 64 SIMT tile kernel would run 64 CTAs for a 4096-row tile).  fp32 FMA,
// like the SIMT path; one instantiation per batch size (no runtime trip
// counts inside the unrolled loops).
//
// forward: acc[b][o] = sum_k W[o][k] x~[b][k].  A warp owns R rows: per
// 16-byte chunk position each lane loads the chunk of all R rows (U chunk
// positions in flight), then every x~ chunk once for all R rows -- the x~
// re-reads through L1 cost (R + B) / R times the W bytes -- and a warp
// reduction at the end.  8 warps per CTA.
constexpr int GV_MAXB = 15;
template <int NB> constexpr int gv_rows() { return NB <= 8 ? 4 : 2; }

template <int NB>
__global__ void __launch_bounds__(256) gemv_fwd_kernel(const float *__restrict__ W, int ldw, int M,
                                                        int K, const float *__restrict__ Xt,
                                                        int ldt, float *__restrict__ acc, int lda,
                                                        const int *__restrict__ n_rows) {
  constexpr int R = gv_rows<NB>();
  if (n_rows && *n_rows != NB) return; // compacted re-issue: one instantiation per count
  const int lane = threadIdx.x & 31;
  const int o0 = (blockIdx.x * 8 + (threadIdx.x >> 5)) * R;
  if (o0 >= M) return;
  float a[R][NB];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int b = 0; b < NB; ++b) a[r][b] = 0.f;
  const float4 *w[R];
#pragma unroll
  for (int r = 0; r < R; ++r)
    w[r] = reinterpret_cast<const float4 *>(W + (size_t)min(o0 + r, M - 1) * ldw);
  const int K4 = K >> 2; // 16-byte chunks (W rows: ld % 32 == 0; x~ rows: ldt % 4 == 0)
  constexpr int U = NB <= 4 ? 4 : 2;
  int c = lane;
  auto step = [&](const float4 (&wv)[R], int cc) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const float4 xv = __ldg(reinterpret_cast<const float4 *>(Xt + (size_t)b * ldt) + cc);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        a[r][b] = fmaf(wv[r].x, xv.x, a[r][b]);
        a[r][b] = fmaf(wv[r].y, xv.y, a[r][b]);
        a[r][b] = fmaf(wv[r].z, xv.z, a[r][b]);
        a[r][b] = fmaf(wv[r].w, xv.w, a[r][b]);
      }
    }
  };
  for (; c + 32 * (U - 1) < K4; c += 32 * U) {
    float4 wv[U][R];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r) wv[u][r] = __ldcs(w[r] + c + 32 * u);
#pragma unroll
    for (int u = 0; u < U; ++u) step(wv[u], c + 32 * u);
  }
  for (; c < K4; c += 32) {
    float4 wv[R];
#pragma unroll
    for (int r = 0; r < R; ++r) wv[r] = __ldcs(w[r] + c);
    step(wv, c);
  }
  for (int k = 4 * K4 + lane; k < K; k += 32) // K % 4 tail
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const float xv = Xt[(size_t)b * ldt + k];
#pragma unroll
      for (int r = 0; r < R; ++r)
        a[r][b] = fmaf(reinterpret_cast<const float *>(w[r])[k], xv, a[r][b]);
    }
#pragma unroll
  for (int b = 0; b < NB; ++b)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const float v = warp_sum(a[r][b]);
      if (lane == 0 && o0 + r < M) acc[(size_t)b * lda + o0 + r] = v;
    }
}

// Fused small-batch forward (B <= 4, no bound management, no input noise):
// the whole noisy MVM in ONE launch.  A CTA of 8 warps owns 32 rows: it
// computes each sample's abs-max alpha (block reduction; the inputs are
// L2-resident), converts K-chunks of the inputs with the DAC into shared
// memory (prep_row's arithmetic; each thread keeps the partial norms of the
// two 512-thread prep threads it stands for and the warp sums are added in
// prep_row's order, so x~ and ||x~|| are bit-identical to the prep kernel's),
// and every warp streams its 4 rows of W against them (16 rows' chunks in
// flight per lane) with every sample's accumulator in registers;
// after a warp reduction lane b runs the output stage (noise, ADC, alpha) of
// sample b.  prep + contraction + epilogue become one W stream.
constexpr int GF_THREADS = 256, GF_ROWS = 4, GF_KC = 4096;
constexpr int GF_MAXB = 2; // larger batches: the staged GEMV path measured faster

template <int NB>
__global__ void __launch_bounds__(GF_THREADS) gemv_fused_fwd_kernel(
    const float *__restrict__ W, int ldw, int M, int K, const float *__restrict__ X, int ldx,
    float *__restrict__ Y, int ldy, IoDev io, Key key, uint64_t seq0, int o0) {
  extern __shared__ float4 xs4[]; // [NB][GF_KC / 4] converted inputs of the chunk
  float *xs = reinterpret_cast<float *>(xs4);
  __shared__ float red[NB][17];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r0 = (blockIdx.x * (GF_THREADS / 32) + warp) * GF_ROWS; // this warp's first row
  {
    // the CTA's rows of W start streaming into L2 now (one bulk prefetch per
    // row), under the abs-max and the DAC below
    const int row = blockIdx.x * (GF_THREADS / 32) * GF_ROWS + threadIdx.x;
    if (threadIdx.x < (GF_THREADS / 32) * GF_ROWS && row < M) {
      const uint32_t bytes = (uint32_t)((K + 3) & ~3) * 4u;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(W + (size_t)row * ldw),
                   "r"(bytes)
                   : "memory");
    }
  }
  // ---- alpha per sample (prep_kernel: block max)
  SampleState st[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    float m = 0.f;
    for (int k = threadIdx.x; k < K; k += GF_THREADS) m = fmaxf(m, fabsf(X[(size_t)b * ldx + k]));
    m = warp_max(m);
    if (lane == 0) red[b][warp] = m;
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    float m = 0.f;
    for (int w2 = 0; w2 < GF_THREADS / 32; ++w2) m = fmaxf(m, red[b][w2]);
    st[b].alpha = (m == 0.f) ? 0.f : (io.nm_absmax ? m : 1.f);
    st[b].m = 0;
    st[b].active = 1;
  }
  __syncthreads();
  // nrm[b][h]: the partial of prep_row's thread threadIdx.x + 256 h
  float nrm[NB][2], a[GF_ROWS][NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    nrm[b][0] = nrm[b][1] = 0.f;
#pragma unroll
    for (int r = 0; r < GF_ROWS; ++r) a[r][b] = 0.f;
  }
  const bool rows_ok = r0 < M;
  const float *w[GF_ROWS];
#pragma unroll
  for (int r = 0; r < GF_ROWS; ++r) w[r] = W + (size_t)min(r0 + r, M - 1) * ldw;
  for (int kc = 0; kc < K; kc += GF_KC) {
    const int n = min(GF_KC, K - kc);
    // ---- DAC of the chunk (prep_row's convert, same thread per element)
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const double inv = st[b].alpha == 0.f ? 0.0 : 1.0 / (double)st[b].alpha;
      const bool fast = !io.perfect && st[b].alpha != 0.f;
      const float a32 = fast ? (float)(inv * pow2i(io.dac.bits) / (2.0 * io.dac.bound)) : 0.f;
      const float c032 = 0.5f * io.dac.flevels_m1;
      const float tie_eps = fast ? __int_as_float((127 + io.dac.bits - 20) << 23) /* 2^(bits-20) */ : 0.f;
      for (int k = threadIdx.x; k < n; k += GF_THREADS) {
        const float xv = X[(size_t)b * ldx + kc + k];
        float f;
        if (io.perfect) {
          f = xv;
        } else if (st[b].alpha == 0.f || xv == 0.f) {
          f = 0.f;
        } else {
          const float t = fmaf(xv, a32, c032);
          const float fr = t - floorf(t);
          if (fabsf(fr - 0.5f) > tie_eps) {
            float kk = floorf(t + 0.5f);
            kk = fminf(fmaxf(kk, 0.f), io.dac.flevels_m1);
            f = fmaf(kk + 0.5f, io.dac.fstep, -io.dac.fbound);
          } else {
            f = (float)quantize((double)xv * inv, io.dac);
          }
        }
        xs[b * GF_KC + k] = f;
        const int h = ((kc + k) >> 8) & 1; // (kc + k) % 512 >= 256
        nrm[b][h] = fmaf(f, f, nrm[b][h]);
      }
    }
    __syncthreads();
    // ---- stream this warp's rows over the chunk
    if (rows_ok) {
      const int n4 = ((n & 3) == 0 && (kc & 3) == 0) ? n >> 2 : 0;
      constexpr int U = NB <= 2 ? 4 : 2;
      for (int c = lane; c < n4; c += 32 * U) {
        float4 wv[U][GF_ROWS];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int r = 0; r < GF_ROWS; ++r)
            wv[u][r] = c + 32 * u < n4 ? __ldcs(reinterpret_cast<const float4 *>(w[r] + kc) + c + 32 * u)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (c + 32 * u >= n4) break;
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            const float4 xv = xs4[b * (GF_KC / 4) + c + 32 * u];
#pragma unroll
            for (int r = 0; r < GF_ROWS; ++r) {
              a[r][b] = fmaf(wv[u][r].x, xv.x, a[r][b]);
              a[r][b] = fmaf(wv[u][r].y, xv.y, a[r][b]);
              a[r][b] = fmaf(wv[u][r].z, xv.z, a[r][b]);
              a[r][b] = fmaf(wv[u][r].w, xv.w, a[r][b]);
            }
          }
        }
      }
      for (int k = 4 * n4 + lane; k < n; k += 32)
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          const float xv = xs[b * GF_KC + k];
#pragma unroll
          for (int r = 0; r < GF_ROWS; ++r) a[r][b] = fmaf(w[r][kc + k], xv, a[r][b]);
        }
    }
    __syncthreads(); // the chunk is read before the next one overwrites it
  }
  // ---- ||x~|| per sample, in prep_row's order: 16 virtual warps of 32
  // (warp w, half h) -> virtual warp 8 h + w
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const float v0 = warp_sum(nrm[b][0]), v1 = warp_sum(nrm[b][1]);
    if (lane == 0) {
      red[b][warp] = v0;
      red[b][8 + warp] = v1;
    }
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    float tot = 0.f;
    for (int w2 = 0; w2 < 16; ++w2) tot += red[b][w2];
    st[b].norm = sqrtf(tot);
  }
  if (!rows_ok) return;
  // ---- every lane gets every sum (butterfly), then lane b finishes sample b
  float mine[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int b = 0; b < NB; ++b)
#pragma unroll
    for (int r = 0; r < GF_ROWS; ++r) {
      const float v = warp_sum(a[r][b]);
      if (lane == b) mine[r] = v;
    }
  if (lane >= NB) return;
  SampleState s = st[0];  // (rows r0 .. r0 + 3: one whole noise group)
#pragma unroll
  for (int b = 1; b < NB; ++b)
    if (lane == b) s = st[b];
  // the warp holds rows r0, r0 + 1 of the 4-row noise group g (o0 % 4 == 0);
  // epilogue_group4 writes only the rows inside [r0, r0 + 2) of this warp
  const int g = (o0 + r0) >> 2;
  epilogue_group4(mine, g, o0, M, s, io, key, seq0 + (uint64_t)lane, Y + (size_t)lane * ldy);
}

// backward: part[s][b][j] = sum over rows i of split s of W[i][j] d~[b][i].
// A thread owns 4 consecutive columns (one 16-byte chunk of a W row: a warp
// reads 512 contiguous bytes per row) and 16 rows in flight; the rows are
// split over blockIdx.y; d~ values are warp-uniform broadcasts.
constexpr int GVB_SPLITS = 64;
template <int NB>
__global__ void __launch_bounds__(128) gemv_bwd_kernel(const float *__restrict__ W, int ldw, int M,
                                                        int K, const float *__restrict__ Dt,
                                                        int ldt, float *__restrict__ part,
                                                        int lda, size_t split_stride,
                                                        int rows_per_split,
                                                        const int *__restrict__ n_rows) {
  if (n_rows && *n_rows != NB) return;
  const int j0 = (blockIdx.x * 128 + threadIdx.x) * 4; // first of this thread's 4 columns
  if (j0 >= M) return;
  const int i0 = blockIdx.y * rows_per_split, i1 = min(K, i0 + rows_per_split);
  float4 a[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) a[b] = make_float4(0.f, 0.f, 0.f, 0.f);
  const bool full = j0 + 3 < M;
  auto ldw4 = [&](int i) {
    const float *row = W + (size_t)i * ldw + j0;
    return full ? __ldcs(reinterpret_cast<const float4 *>(row))
                : make_float4(row[0], j0 + 1 < M ? row[1] : 0.f, j0 + 2 < M ? row[2] : 0.f, 0.f);
  };
  auto fma4 = [&](const float4 &wv, int i) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const float dv = __ldg(Dt + (size_t)b * ldt + i);
      a[b].x = fmaf(wv.x, dv, a[b].x);
      a[b].y = fmaf(wv.y, dv, a[b].y);
      a[b].z = fmaf(wv.z, dv, a[b].z);
      a[b].w = fmaf(wv.w, dv, a[b].w);
    }
  };
  int i = i0;
  constexpr int U = NB <= 4 ? 16 : 8;
  for (; i + U <= i1; i += U) {
    float4 wv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) wv[u] = ldw4(i + u);
#pragma unroll
    for (int u = 0; u < U; ++u) fma4(wv[u], i + u);
  }
  for (; i < i1; ++i) fma4(ldw4(i), i);
  float *dst = part + (size_t)blockIdx.y * split_stride;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    float *o = dst + (size_t)b * lda + j0;
    if (full && ((lda & 3) == 0)) {
      *reinterpret_cast<float4 *>(o) = a[b];
    } else {
      o[0] = a[b].x;
      if (j0 + 1 < M) o[1] = a[b].y;
      if (j0 + 2 < M) o[2] = a[b].z;
      if (j0 + 3 < M) o[3] = a[b].w;
    }
  }
}

// out[e] = sum_{s < S} part[s][e] in split order (e < n): the backward
// GEMV's row splits, reduced with one thread per element
// (16 loads in flight per thread, summed in split order; small CTAs spread
// the few thousand elements of a per-sample call over many SMs)
__global__ void __launch_bounds__(64) split_reduce_kernel(const float *__restrict__ part, int S,
                                                           size_t stride, size_t n,
                                                           float *__restrict__ out) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n;
       e += (size_t)gridDim.x * blockDim.x) {
    float v = 0.f;
    int s = 0;
    for (; s + 16 <= S; s += 16) {
      float t[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) t[u] = __ldcg(part + (size_t)(s + u) * stride + e);
#pragma unroll
      for (int u = 0; u < 16; ++u) v = (s + u == 0) ? t[u] : v + t[u];
    }
    for (; s < S; ++s) v = (s == 0) ? part[e] : v + part[(size_t)s * stride + e];
    out[e] = v;
  }
}

// --------------------------------------------------------------- epilogue
// one thread = one group of 4 outputs of one sample (xb_mvm_common.cuh).
// acc row r (r < n; n = *n_rows for a compacted re-issue) holds sample
// map[r] (re-issue) or n0 + r (pass 0); rows of one N slab per launch.
__global__ void __launch_bounds__(256) epilogue_kernel(const float *__restrict__ acc, int lda,
                                                        int nsplit, size_t split_stride, int M,
                                                        int o0, float *__restrict__ Y, int ldy,
                                                        const SampleState *__restrict__ st,
                                                        IoDev io, Key key, uint64_t seq0,
                                                        BmBufs bm, int nb, int n0, int pass,
                                                        const int *__restrict__ map,
                                                        const int *__restrict__ n_rows) {
  const int row = blockIdx.y;
  if (n_rows && row >= *n_rows) return;
  const int b = map ? map[row] : n0 + row;
  const SampleState s = st[b];
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
  bm_flag(hit, s, io, bm.flags + (pass & 1) * nb + (b - n0));
}

// Row-shard backward, phase 1: the shard's column sums plus its share of the
// weight-noise fold (independent per shard: the variances of the shards add
// up to sigma_w^2 ||d~||^2 over all rows).  No output noise, ADC or alpha yet.
__global__ void __launch_bounds__(256) partial_kernel(const float *__restrict__ acc, int M,
                                                       int nsplit, size_t split_stride,
                                                       float *__restrict__ P,
                                                       const SampleState *__restrict__ st,
                                                       IoDev io, Key key, uint64_t seq0,
                                                       uint32_t shard_tag, int B) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= M) return;
  for (int b = blockIdx.y; b < B; b += gridDim.y) { // (gridDim.y <= 65535)
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
}

// Row-shard backward, phase 2 (after the sum over shards): output noise, ADC
// and alpha act on the reduced column sums, as in proj/src/io.cpp:143-146.
// Same noise groups as epilogue_kernel (o0 = 0, m = 0), so the split-phase
// backward reproduces the whole-tile backward bit for bit.
__global__ void __launch_bounds__(256) finish_kernel(const float *__restrict__ Psum, int M,
                                                      const float *__restrict__ amax,
                                                      float *__restrict__ Y, IoDev io, Key key,
                                                      uint64_t seq0, int B) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (4 * g >= M) return;
  io.sigma_w = 0.0;
  for (int b = blockIdx.y; b < B; b += gridDim.y) { // (gridDim.y <= 65535)
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
  // words and arithmetic as the whole-tile output stage (sigma_w = 0 above)
  epilogue_group4(a, g, 0, M, s, io, key, seq0 + (uint64_t)b, Y + (size_t)b * M);
  }
}

struct MvmScratch {
  float *xt;
  float *xt1;   // x~ at m = 1 [B][ldt] (in-kernel bound management), else null
  SampleState *st1;
  float *acc;   // pass 0 partial sums [nsplit][B][M] (unfused)
  float *acc_r; // re-issue partial sums [nsplit][256][M] (unfused)
  SampleState *st;
  int *bm;      // per slab: flags [2][256], counts [64]; then grid barriers [nslab]
  int *map;     // [B]
  int bm_words;
};

constexpr int SLAB = 256;

MvmScratch carve(Tile &t, int B, int K, int M, int nsplit, bool level1) {
  const int nslab = (B + SLAB - 1) / SLAB;
  const size_t xt_b = (size_t)B * K * sizeof(float);
  const size_t xt1_b = level1 ? xt_b : 0, st1_b = level1 ? (size_t)B * sizeof(SampleState) : 0;
  const size_t acc_b = (size_t)nsplit * B * M * sizeof(float);
  const size_t accr_b = nsplit ? (size_t)nsplit * std::min(B, SLAB) * M * sizeof(float) : 0;
  const size_t st_b = (size_t)B * sizeof(SampleState);
  const int bm_words = nslab * (BM_SLAB_WORDS + 1);
  const size_t bm_b = (size_t)bm_words * sizeof(int);
  const size_t map_b = (size_t)B * sizeof(int);
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  char *p = (char *)t.s_io.get(al(xt_b) + al(acc_b) + al(accr_b) + al(st_b) + al(bm_b) +
                               al(map_b) + al(xt1_b) + al(st1_b));
  MvmScratch s;
  s.xt = (float *)p;
  p += al(xt_b);
  s.xt1 = level1 ? (float *)p : nullptr;
  p += al(xt1_b);
  s.st1 = level1 ? (SampleState *)p : nullptr;
  p += al(st1_b);
  s.acc = (float *)p;
  p += al(acc_b);
  s.acc_r = (float *)p;
  p += al(accr_b);
  s.st = (SampleState *)p;
  p += al(st_b);
  s.bm = (int *)p;
  p += al(bm_b);
  s.map = (int *)p;
  s.bm_words = bm_words;
  return s;
}

BmBufs slab_bufs(const MvmScratch &s, int slab) {
  BmBufs b;
  b.flags = s.bm + (size_t)slab * BM_SLAB_WORDS;
  b.counts = b.flags + 2 * SLAB;
  b.map = s.map + (size_t)slab * SLAB;
  return b;
}

template <bool TRANS>
void gemm(Tile &t, const float *xt, int ldt, int M, int K, int B, float *acc,
          const int *n_rows) {
  dim3 grid((M + 63) / 64, (B + 63) / 64);
  mvm_simt_kernel<TRANS><<<grid, 256, 0, t.stream>>>(t.W, t.ld, M, K, xt, ldt, B, acc, M, n_rows);
  count_launch();
  XB_CUDA(cudaGetLastError());
}

// the fused small-batch forward (one launch: DAC, contraction, output stage)
static void gemv_fused_fwd(Tile &t, const float *X, int K, int M, int B, float *Y, IoDev io,
                           Key key, uint64_t seq0, int o0) {
  io.exact = 1; // the exact fp32 path's output stage (fp64 converters)
  constexpr int rows_per_cta = (GF_THREADS / 32) * GF_ROWS;
  dim3 g((M + rows_per_cta - 1) / rows_per_cta);
#define XB_GF(NB)                                                                          \
  case NB: {                                                                               \
    const int smem = NB * GF_KC * (int)sizeof(float);                                      \
    static std::atomic<uint64_t> cfg_##NB{0};                                              \
    once_per_device(cfg_##NB, [&] {                                                        \
      XB_CUDA(cudaFuncSetAttribute(gemv_fused_fwd_kernel<NB>,                              \
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, smem));    \
    });                                                                                    \
    gemv_fused_fwd_kernel<NB><<<g, GF_THREADS, smem, t.stream>>>(t.W, t.ld, M, K, X, K, Y, M, \
                                                                 io, key, seq0, o0);       \
    break;                                                                                 \
  }
  switch (B) {
    XB_GF(1) XB_GF(2)
  }
#undef XB_GF
  count_launch();
  XB_CUDA(cudaGetLastError());
}

// The small-batch contraction (B <= GV_MAXB) into acc [B][M] (lda = M).
// The backward stages its row-split partials in `work` ([S][B][M], S =
// GVB_SPLITS) and reduces them in order; a compacted re-issue (n_rows on
// the device) runs the instantiation of every batch size up to B, each of
// which leaves unless it matches the count.
template <bool TRANS>
void gemv(Tile &t, const float *xt, int ldt, int M, int K, int B, float *acc, float *work,
          const int *n_rows) {
  const int lo = n_rows ? 1 : B;
  for (int nb = lo; nb <= B; ++nb) {
#define XB_GV(NB)                                                                            case NB:                                                                                     if (TRANS) {                                                                                 const int rps = (K + GVB_SPLITS - 1) / GVB_SPLITS;                                         dim3 g((M + 511) / 512, (K + rps - 1) / rps);                                              gemv_bwd_kernel<NB><<<g, 128, 0, t.stream>>>(t.W, t.ld, M, K, xt, ldt, work, M,                                                         (size_t)NB * M, rps, n_rows);                  count_launch();                                                                            split_reduce_kernel<<<std::min<size_t>(((size_t)NB * M + 63) / 64, 8192), 64, 0,                              t.stream>>>(work, (int)g.y, (size_t)NB * M, (size_t)NB * M, acc);     } else {                                                                                     dim3 g((M + 8 * gv_rows<NB>() - 1) / (8 * gv_rows<NB>()));                                 gemv_fwd_kernel<NB><<<g, 256, 0, t.stream>>>(t.W, t.ld, M, K, xt, ldt, acc, M, n_rows);     }                                                                                          break;
    switch (nb) {
      XB_GV(1) XB_GV(2) XB_GV(3) XB_GV(4) XB_GV(5) XB_GV(6) XB_GV(7) XB_GV(8)
      XB_GV(9) XB_GV(10) XB_GV(11) XB_GV(12) XB_GV(13) XB_GV(14) XB_GV(15)
    }
#undef XB_GV
    count_launch();
    XB_CUDA(cudaGetLastError());
  }
}


// XB_MVM_UNFUSED=1 forces the split-K partials + epilogue kernel path: the
// parity tests run both and require bit-identical outputs
static bool unfused_requested() {
  const char *e = getenv("XB_MVM_UNFUSED");
  return e && e[0] == '1';
}
// XB_BM_HOST_PASSES=1 forces host-driven re-issue passes on the fused path
// (the sharded mode; tests compare it with the in-kernel loop)
static bool host_passes_requested() {
  const char *e = getenv("XB_BM_HOST_PASSES");
  return e && e[0] == '1';
}

// XB_BM_NO_LEVEL1=1: every in-kernel re-issue is compacted and prepared after
// its barrier (A/B measurements of the prestaged m = 1 slab)
static bool level1_disabled() {
  const char *e = getenv("XB_BM_NO_LEVEL1");
  return e && e[0] == '1';
}

// tensor-core contraction at TF32 / 3xTF32 (B >= 16); the fp32 SIMT kernel
// otherwise (exact-fp32 parity mode, tiny batches)
static bool use_tc(const Tile &t, int B) {
  return (t.cfg.mvm_precision == XB_MVM_TF32 || t.cfg.mvm_precision == XB_MVM_TF32X3) && B >= 16;
}

// One full noisy MVM in direction TRANS (forward: false).  Nothing here waits
// on the device:
//  * pass 0: prep (alpha, x~, norms; clears the BM buffers) + contraction with
//    the output stage;
//  * bound management, tensor cores, unsharded: the re-issue passes run inside
//    the contraction launch (grid barriers between passes);
//  * otherwise (SIMT, unfused, row shards, or a grid that cannot be
//    co-resident): bm_max_iter re-issue passes are enqueued per N slab --
//    compaction, prep, contraction, output stage -- each of which leaves at
//    once when the previous pass flagged nothing.  Row shards all-reduce the
//    flags (max) before every compaction, so every shard re-issues exactly
//    the samples the unsharded tile would.
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
  const int in0 = TRANS ? t.row0 : 0; // global index of input 0 (input-noise counters)
  // the output stage runs inside the tcgen05 kernel (K-splits reduced over a
  // thread-block cluster) unless the caller wants raw partial sums, the noise
  // groups of 4 outputs do not align with the tile, or a cluster would exceed
  // the portable 8 CTAs (both paths use the same K-splits: bit-identical)
  const int splits = tc ? tc_used_splits(K, std::min(8, tc_splits(M, K, x3))) : 1;
  const bool fused = tc && !skip_epilogue && (o0 & 3) == 0 && !unfused_requested();
  const int ldt = (K + 3) & ~3; // x~ rows padded to 16 bytes (TMA global stride)
  // small batches on the exact fp32 path stream W once (GEMV); the backward
  // GEMV splits the rows (partials summed in order by the epilogue kernel)
  const bool gv = !tc && B <= GV_MAXB;
  // (GEMV backward: acc_r holds the row-split partials; GVB_SPLITS sets of B x M)
  const bool bm = io.bm && !skip_epilogue;
  const bool sharded_bm = bm && t.comm && !TRANS;
  const bool want_loop = fused && bm && !sharded_bm && !host_passes_requested();
  // the loop's first re-issue streams an m = 1 slab the contraction's idle
  // warps prepare during pass 0 (FusedOut::xt1; TF32: 3xTF32 has no idle warps)
  const bool level1 = want_loop && !x3 && io.bm_max_iter >= 1 && !level1_disabled();
  MvmScratch s = carve(t, B, ldt, M, fused ? 0 : (tc ? splits : (gv && TRANS ? GVB_SPLITS : 1)),
                       level1);
  const int nslab = (B + SLAB - 1) / SLAB;
  int *bars = s.bm + (size_t)nslab * BM_SLAB_WORDS;

  // small batches without bound management or input noise: the whole MVM in
  // one launch (DAC on the fly, output stage fused; gemv_fused_fwd_kernel)
  const bool dac_fast = io.perfect || (io.dac.bits > 0 && io.dac.bits <= 16 && io.dac.pow2);
  if (gv && B <= GF_MAXB && !TRANS && !bm && !skip_epilogue && io.sigma_inp == 0.0 && dac_fast &&
      (o0 & 3) == 0 && !amax_in && !unfused_requested()) {
    gemv_fused_fwd(t, dIn, K, M, B, dOut, io, key, seq0, o0);
    return;
  }
  prep_kernel<<<B, PREP_THREADS, 0, t.stream>>>(dIn, K, s.xt, ldt, s.st, io, key, seq0, amax_in,
                                                 in0, bm ? s.bm : nullptr, s.bm_words);
  count_launch();
  XB_CUDA(cudaGetLastError());

  FusedOut fo{};
  fo.Y = dOut;
  fo.ldy = M;
  fo.st = s.st;
  fo.io = io;
  fo.key = key;
  fo.seq0 = seq0;
  fo.bm = slab_bufs(s, 0);
  fo.pass = 0;
  fo.o0 = o0;
  fo.X = dIn;
  fo.K = K;
  fo.in0 = in0;
  fo.xt = s.xt;
  fo.ldt = ldt;
  fo.bar = reinterpret_cast<unsigned *>(bars);
  fo.xt1 = s.xt1;
  fo.st1 = s.st1;

  // ---- pass 0
  bool looped = false;
  int nsplit = 1;
  if (fused) {
    looped = tc_gemm(t, TRANS, x3, s.xt, ldt, B, nullptr, splits, &fo, nullptr, want_loop);
  } else if (tc) {
    tc_gemm(t, TRANS, x3, s.xt, ldt, B, s.acc, splits, nullptr);
    nsplit = splits;
  } else if (gv) {
    gemv<TRANS>(t, s.xt, ldt, M, K, B, s.acc, s.acc_r, nullptr);
  } else {
    gemm<TRANS>(t, s.xt, ldt, M, K, B, s.acc, nullptr);
  }
  if (skip_epilogue) { // row shard: partial sums + this shard's weight-noise fold
    dim3 eg((M + 255) / 256, std::min(B, 65535));
    partial_kernel<<<eg, 256, 0, t.stream>>>(s.acc, M, nsplit, (size_t)B * M, dPartial, s.st,
                                             io, key, seq0,
                                             (TAG_W_NOISE << 24) | (uint32_t)t.row0, B);
    count_launch();
    XB_CUDA(cudaGetLastError());
    return;
  }
  if (!fused) {
    for (int sl = 0; sl < nslab; ++sl) {
      const int n0 = sl * SLAB, nb = std::min(SLAB, B - n0);
      dim3 eg((out_groups(o0, M) + 255) / 256, nb);
      epilogue_kernel<<<eg, 256, 0, t.stream>>>(s.acc + (size_t)n0 * M, M, nsplit,
                                                (size_t)B * M, M, o0, dOut, M, s.st, io, key,
                                                seq0, slab_bufs(s, sl), nb, n0, 0, nullptr,
                                                nullptr);
      count_launch();
      XB_CUDA(cudaGetLastError());
    }
  }
  if (!bm || looped) return;

  // ---- host-driven re-issue passes (enqueued; each leaves early when idle)
  for (int pass = 1; pass <= io.bm_max_iter; ++pass) {
    for (int sl = 0; sl < nslab; ++sl) {
      const int n0 = sl * SLAB, nb = std::min(SLAB, B - n0);
      BmBufs bb = slab_bufs(s, sl);
      if (sharded_bm) // every shard re-issues the samples saturated on ANY shard
        t.comm->allreduce_max_i32(bb.flags + ((pass - 1) & 1) * nb, nb, t.stream);
      int *cnt = bb.counts + 32 + pass;
      compact_kernel<<<1, 256, 0, t.stream>>>(bb.flags, nb, n0, pass - 1, bb.map, cnt);
      count_launch();
      float *xt = s.xt + (size_t)n0 * ldt; // the slab's x~ rows, compacted from row 0
      reprep_kernel<<<nb, PREP_THREADS, 0, t.stream>>>(dIn, K, xt, ldt, s.st, io, key, seq0, in0,
                                                       bb.map, cnt);
      count_launch();
      XB_CUDA(cudaGetLastError());
      if (fused) { // one slab: its x~ rows, BM buffers and first sample
        FusedOut f = fo;
        f.bm = bb;
        f.pass = pass;
        f.n_dev = cnt;
        f.n0 = n0;
        f.xt = xt;
        f.loop = 0;
        tc_gemm(t, TRANS, x3, xt, ldt, nb, nullptr, splits, &f);
      } else {
        float *acc = tc ? s.acc_r : s.acc;
        int ns = 1;
        if (tc) {
          tc_gemm(t, TRANS, x3, xt, ldt, nb, acc, splits, nullptr, cnt);
          ns = splits;
        } else if (gv) {
          gemv<TRANS>(t, xt, ldt, M, K, nb, s.acc, s.acc_r, cnt);
          acc = s.acc;
        } else {
          gemm<TRANS>(t, xt, ldt, M, K, nb, acc, cnt);
        }
        dim3 eg((out_groups(o0, M) + 255) / 256, nb);
        epilogue_kernel<<<eg, 256, 0, t.stream>>>(acc, M, ns, (size_t)nb * M, M, o0,
                                                  dOut, M, s.st, io, key, seq0, bb, nb, n0, pass,
                                                  bb.map, cnt);
        count_launch();
        XB_CUDA(cudaGetLastError());
      }
    }
  }
}

} // namespace

// ---- Tiki-Taka transfer read (compound.cpp:257-267) -----------------------
// The forward of the one-hot e_col (B = 1, the exact fp32 path): prep gives
// alpha = max|e_col| = 1, x~ = Q_dac(e_col) -- zero except Q_dac(1) at col,
// exact zeros pass the quantizer -- and ||x~|| = |Q_dac(1)|; every fp32 sum of
// the contraction then reduces to the one product W[i][col] Q_dac(1).  So the
// read is a strided gather of one column and the shared output stage (same
// noise counters, fp64 converters): bit-identical to the full forward, at R
// loads instead of a pass over the whole tile.
__global__ void __launch_bounds__(256) column_read_kernel(const float *__restrict__ W, int ld, int R,
                                                           int C, int col, IoDev io, Key key,
                                                           uint64_t seq, float *__restrict__ out,
                                                           float *__restrict__ onehot) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int k = tid; k < C; k += gridDim.x * blockDim.x) onehot[k] = k == col ? 1.f : 0.f;
  const int g = tid;
  if (4 * g >= R) return;
  const float xq = io.perfect ? 1.f : (float)quantize(1.0, io.dac);
  SampleState s;
  s.alpha = 1.f;
  s.m = 0;
  s.active = 1;
  s.norm = sqrtf(fmaf(xq, xq, 0.f));
  float a[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int row = 4 * g + k;
    a[k] = row < R ? W[(size_t)row * ld + col] * xq : 0.f;
  }
  epilogue_group4(a, g, 0, R, s, io, key, seq, out);
}

void launch_column_read(Tile &t, int col, const IoDev &io_in, Key key, uint64_t seq, float *out,
                        float *onehot) {
  IoDev io = io_in;
  io.exact = 1; // a single sample takes the exact fp32 path (fp64 converters)
  const int n = std::max((t.R + 3) / 4, (t.C + 3) / 4);
  column_read_kernel<<<(n + 255) / 256, 256, 0, t.stream>>>(t.W, t.ld, t.R, t.C, col, io, key,
                                                            seq, out, onehot);
  count_launch();
  XB_CUDA(cudaGetLastError());
}

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
  dim3 eg((out_groups(0, t.C) + 255) / 256, std::min(B, 65535));
  finish_kernel<<<eg, 256, 0, t.stream>>>(dPsum, t.C, amax_global, dG, io2, key, seq0, B);
  count_launch();
  XB_CUDA(cudaGetLastError());
}

} // namespace xb
