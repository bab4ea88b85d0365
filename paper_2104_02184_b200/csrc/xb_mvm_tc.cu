// xb_mvm_tc.cu -- the MVM contraction on the 5th-generation tensor cores.
//
// acc[s][b][o] = sum_{k in split s} W[o][k] x~[b][k]  (forward, both operands K-major)
//
// One CTA = one 128-row tile of W (M) x all BN <= 256 samples (N) x one
// K-split.  TMA (cp.async.bulk.tensor, 128-byte swizzle) streams 32-wide K
// blocks of W and x~ into a 4-stage shared-memory ring; a single thread
// issues tcgen05.mma.kind::tf32 (M=128, N=BN, K=8, four per stage) into a
// TMEM accumulator of BN fp32 columns; mbarriers chain TMA -> MMA -> smem
// release (tcgen05.commit) and MMA -> epilogue.  The four warps then drain
// TMEM with tcgen05.ld (warp w owns accumulator lanes 32w..32w+31 = output
// rows).
//
// Fused epilogue (FUSED): the K-splits of one M-tile form a thread-block
// cluster.  Each CTA parks its partial tile in its own shared memory, and
// after a cluster barrier CTA r reduces columns (samples) [r n/S, (r+1) n/S)
// over the S partials through distributed shared memory (mapa +
// ld.shared::cluster) and applies the output stage -- sigma_w fold, output
// noise, ADC, alpha 2^m, bound-management flags (xb_mvm_common.cuh) --
// writing Y directly.  No partial sums touch HBM and no epilogue kernel runs.
// Unfused: the partial sums go to HBM for epilogue_kernel / the row-shard
// split-phase backward.
//
// W is row-major [R][ld] fp32, x~ is [B][K] fp32 -- the kernel reads the same
// bytes the SIMT path reads; the tensor core consumes them as TF32.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "xb_mvm_common.cuh"

#ifdef XB_TC_TRACE
// experiment builds only: per-CTA globaltimer stamps of the contraction
// (start, first stage landed, accumulator complete, end)
__device__ unsigned long long g_tc_trace[4096][16];
__device__ __forceinline__ unsigned long long xb_gtime() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  return v;
}
#define XB_TRACE(k)                                                                             \
  do {                                                                                          \
    const unsigned slot_ = blockIdx.x + gridDim.x * blockIdx.y;                                 \
    if (slot_ < 4096) g_tc_trace[slot_][k] = xb_gtime();                                        \
  } while (0)
extern "C" __attribute__((visibility("default"))) int xb_debug_tc_trace(unsigned long long *out,
                                                                          int n) {
  return (int)cudaMemcpyFromSymbol(out, g_tc_trace, sizeof(unsigned long long) * 16 *
                                                        (size_t)(n < 4096 ? n : 4096));
}
#else
#define XB_TRACE(k) ((void)0)
#endif

namespace xb {

namespace {

constexpr int TC_BM = 128; // rows of one UMMA (M) = one TMEM lane per row
constexpr int TC_BK = 32;  // fp32 elements per 128-byte swizzle row
constexpr int TC_MAX_BN = 256;
constexpr int TC_A_BYTES = TC_BM * TC_BK * 4;     // 16 KB per 128-row sub-tile
constexpr int TC_B_BYTES = TC_MAX_BN * TC_BK * 4; // 32 KB (max)
// A CTA owns NSUB 128-row sub-tiles of the output (NSUB accumulators of BN
// TMEM columns) and streams ONE x~ tile per K-block for all of them: the
// x~ operand is re-read once per CTA row-band, so NSUB = 2 halves its L2->SM
// traffic (x~ is the larger operand per K-block at N = 256 > M = 128).
// TF32: ring of (A, B); 3xTF32: 2-stage ring of (A_hi, B_hi, A_lo, B_lo).
template <bool X3, int NSUB> constexpr int tc_stage_bytes() {
  return (X3 ? 2 : 1) * (NSUB * TC_A_BYTES + TC_B_BYTES);
}
template <bool X3, int NSUB> constexpr int tc_stages() {
  return X3 ? 2 : (NSUB == 1 ? 4 : 3);
}
template <bool X3, int NSUB> constexpr int tc_smem() {
  return tc_stages<X3, NSUB>() * tc_stage_bytes<X3, NSUB>() + 1024 /*align*/ + 256 /*bars*/;
}
// threads: 128 = producer warp, MMA warp, two more epilogue warps; 3xTF32
// adds converter warps; the fused output stage wants more warps in flight
#ifndef XB_TC_FUSED_THREADS
#define XB_TC_FUSED_THREADS 512
#endif
template <bool X3, bool FUSED = false> constexpr int tc_threads() {
  return FUSED ? XB_TC_FUSED_THREADS : (X3 ? 256 : 128);
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "XB_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra XB_WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, uint32_t bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

// UMMA shared-memory descriptor, sm_100 version 1.
//  K-major (layout 2 = SWIZZLE_128B): 8-row groups of 128-byte rows, SBO = 1024 B
//    between groups (LBO unused)
//  MN-major tf32 (layout 1 = SWIZZLE_128B_BASE32B, the only MN-major layout the
//    tensor core accepts for 32-bit operands): atoms of 32 MN-elements x 4 K-rows
//    (512 B, 32-byte swizzle granule); SBO = 512 B between K-groups, LBO =
//    distance between 32-wide MN atoms
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);   // start address
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16; // leading byte offset
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32; // stride byte offset
  d |= (uint64_t)1u << 46;                   // descriptor version (sm_100)
  d |= (uint64_t)layout << 61;
  return d;
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, B K-major, A K- or
// MN-major, M=128, N=bn
__host__ __device__ __forceinline__ uint32_t idesc_tf32(int bn, bool a_mn = false) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) |
         ((uint32_t)(bn >> 3) << 17) | ((uint32_t)(TC_BM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}

#define XB_TMEM_LD32(taddr, r)                                                                  \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 "                                       \
               "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"                       \
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"      \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),        \
                 "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),      \
                 "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]),  \
                 "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),  \
                 "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),  \
                 "=r"(r[30]), "=r"(r[31])                                                      \
               : "r"(taddr))

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
  uint32_t n;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(n));
  return n;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// address of the same shared-memory word in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t dsmem_map(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}


// split x into hi = x with the low 13 mantissa bits cleared (exactly a TF32
// value, so the tensor core reads it unchanged whether it truncates or
// rounds) and lo = x - hi (exact in fp32; TF32-rounded by the MMA)
__device__ __forceinline__ void split_tf32(float4 &v, float4 &lo) {
  float *e = reinterpret_cast<float *>(&v), *l = reinterpret_cast<float *>(&lo);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const float hi = __uint_as_float(__float_as_uint(e[c]) & 0xffffe000u);
    l[c] = e[c] - hi;
    e[c] = hi;
  }
}

__device__ __forceinline__ float4 dsmem_ld4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}

// Cluster-fused output stage (split-K reduction over distributed shared
// memory).  Every warp of the CTA drains this CTA's accumulator (NSUB
// sub-tiles of 128 TMEM lanes x bnr columns) into its idle pipeline memory
// as [bnr][128] fp32 (tcgen05.ld, lane = row: conflict-free stores); after a
// cluster barrier CTA r reduces columns (samples) [r c, (r + 1) c) over the
// S split partials -- split q lives in cluster CTA q -- through distributed
// shared memory (mapa + ld.shared::cluster.v4, all S loads in flight, summed
// in split order like the epilogue kernel, so fused and unfused agree bit
// for bit) and runs the output stage (xb_mvm_common.cuh) straight into Y.
// (Measured on B200, 4096^2 x 256: pushing the partials to their owners with
// st.shared::cluster instead -- scalar or 16-byte scattered -- was slower:
// DSMEM moves whole-warp contiguous lines best, which the pull form keeps.)
// (Measured alternative, round 2: staging the partials in L2 and reading them
// back with ld.global.cg was slower still -- the drain to global memory alone
// took 4 us vs 1.5 us into shared memory.)
// Column loop of the fused output stage: thread = group of 4 rows (grp) x
// every NW-th column of this CTA's range.  Software-pipelined: the S partial
// loads of the next column (all in flight) are issued before the output
// stage of the current one, so the ~20 B/clk DSMEM stream overlaps the math.
template <int NW, int NS>
__device__ __forceinline__ void reduce_columns(const FusedOut &fo, const float *red,
                                               uint32_t red_s, int row0, int M, int c_lo,
                                               int c_hi, uint32_t my_split, uint32_t nsplit,
                                               const int *map, const SampleState *st,
                                               const int *live, int *flags) {
  const int grp = threadIdx.x & 31, cph = threadIdx.x >> 5;
  auto load = [&](int c, float4 (&v)[NS]) {
    const uint32_t off = red_s + (uint32_t)((c * TC_BM + 4 * grp) * 4);
#pragma unroll
    for (int r = 0; r < NS; ++r)
      if (r < (int)nsplit)
        v[r] = r == (int)my_split ? *reinterpret_cast<const float4 *>(red + (off - red_s) / 4)
                                  : dsmem_ld4(dsmem_map(off, (uint32_t)r));
  };
  // the column's sample, its state and (first prestaged re-issue) whether
  // the previous pass flagged it: loaded one column ahead with the partials
  auto meta = [&](int c, int &b, SampleState &sst, bool &on) {
    b = map ? map[c] : fo.n0 + c;
    on = !live || live[c] != 0;
    sst = st[b];
  };
  int c = c_lo + cph;
  if (c >= c_hi) return;
  float4 v[NS];
  load(c, v);
  int b;
  SampleState sst;
  bool on;
  meta(c, b, sst, on);
  const bool rows_ok = row0 + 4 * grp < M;
  for (;;) {
    const int cn = c + NW;
    float4 vn[NS];
    int bn_ = 0;
    SampleState sn{};
    bool onn = false;
    if (cn < c_hi) {
      if (NS <= 4) load(cn, vn); // (8 splits: no registers to spare)
      meta(cn, bn_, sn, onn);
    }
    float4 acc4 = v[0];
#pragma unroll
    for (int r = 1; r < NS; ++r) // split order (as the epilogue kernel)
      if (r < (int)nsplit) {
        acc4.x += v[r].x;
        acc4.y += v[r].y;
        acc4.z += v[r].z;
        acc4.w += v[r].w;
      }
    if (rows_ok && on) {
      const float a[4] = {acc4.x, acc4.y, acc4.z, acc4.w};
      // global output index of this group: o0 + row0 + 4 grp (o0 % 4 == 0 on
      // the fused path, so groups align with the noise groups)
      const int g = (fo.o0 + row0) / 4 + grp;
      const bool hit = epilogue_group4(a, g, fo.o0, M, sst, fo.io, fo.key,
                                       fo.seq0 + (uint64_t)b, fo.Y + (size_t)b * fo.ldy);
      bm_flag(hit, sst, fo.io, flags + (b - fo.n0));
    }
    if (cn >= c_hi) break;
    if (NS <= 4) {
#pragma unroll
      for (int r = 0; r < NS; ++r) v[r] = vn[r];
    } else {
      load(cn, v);
    }
    c = cn;
    b = bn_;
    sst = sn;
    on = onn;
  }
}

// The m = 1 x~ rows of the slab (FusedOut::xt1/st1), prepared by the warps
// idle during pass 0's mainloop (warps 2.., TF32), sample c on CTA c mod grid.
// Bit-identical to prep_row run by XB_PREP_THREADS threads: each helper warp
// plays whole virtual warps of that block -- virtual thread t converts
// j = t + XB_PREP_THREADS u in ascending u and sums the squares in that
// order -- and the 16 warp sums are added in virtual-warp order.
__device__ __forceinline__ void stage_level1(const FusedOut &fo, float *red) {
  constexpr int VW = XB_PREP_THREADS / 32;
  const int hw = (int)(threadIdx.x >> 5) - 2, nh = (int)(blockDim.x >> 5) - 2;
  const int lane = threadIdx.x & 31;
  const unsigned cta = blockIdx.x + gridDim.x * blockIdx.y, nctas = gridDim.x * gridDim.y;
  const int K = fo.K;
  for (int c = (int)cta; c < fo.nb; c += (int)nctas) {
    const int b = fo.n0 + c;
    SampleState s = fo.st[b];
    s.m = 1;
    const RowDac dac(s, fo.io);
    const uint64_t seq = fo.seq0 + (uint64_t)b;
    const float *x = fo.X + (size_t)b * K;
    float *xt = fo.xt1 + (size_t)c * fo.ldt;
    for (int vw = hw; vw < VW; vw += nh) {
      const int t = vw * 32 + lane;
      float nrm = 0.f;
      for (int j0 = 0; j0 < K; j0 += XB_PREP_THREADS * PREP_VPT) {
        float v[PREP_VPT];
#pragma unroll
        for (int u = 0; u < PREP_VPT; ++u) {
          const int j = j0 + t + u * XB_PREP_THREADS;
          v[u] = j < K ? x[j] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < PREP_VPT; ++u) {
          const int j = j0 + t + u * XB_PREP_THREADS;
          if (j < K) {
            const float f = dac(v[u], j, s, fo.io, fo.key, seq, fo.in0);
            xt[j] = f;
            nrm = fmaf(f, f, nrm);
          }
        }
      }
      nrm = warp_sum(nrm);
      if (lane == 0) red[vw] = nrm;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(nh * 32) : "memory");
    if (hw == 0 && lane == 0) {
      float tot = 0.f;
      for (int w = 0; w < VW; ++w) tot += red[w];
      s.norm = sqrtf(tot);
      fo.st1[b] = s;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(nh * 32) : "memory");
  }
  // pass 1 streams these rows with TMA (async proxy), after the grid barrier
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <int NW, int NSUB>
__device__ __forceinline__ void fused_output_stage(const FusedOut &fo, uint32_t tmem,
                                                   uint8_t *smem, int nkb, int m0, int M, int n,
                                                   int bnr, uint32_t my_split, uint32_t nsplit,
                                                   const int *map, int pass, bool level1) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, quarter = warp & 3;
  float *red = reinterpret_cast<float *>(smem);
  const uint32_t red_s = smem_u32(red);
  const int cols = (bnr + (int)nsplit - 1) / (int)nsplit;
  const int c_lo = (int)my_split * cols, c_hi = min(n, c_lo + cols);
  int *flags = fo.bm.flags + (pass & 1) * fo.nb;
  // prestaged m = 1 pass: every column of the slab, written where pass 0 flagged
  const SampleState *st = level1 ? fo.st1 : fo.st;
  const int *live = level1 ? fo.bm.flags + ((pass - 1) & 1) * fo.nb : nullptr;
#pragma unroll 1
  for (int sub = 0; sub < NSUB; ++sub) {
    const int row = quarter * 32 + lane;
    for (int c0 = 32 * (warp >> 2); c0 < bnr; c0 += 32 * (NW / 4)) {
      uint32_t r[32];
      XB_TMEM_LD32(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(sub * TC_MAX_BN + c0), r);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int c = 0; c < 32; ++c) red[(c0 + c) * TC_BM + row] = nkb > 0 ? __uint_as_float(r[c]) : 0.f;
    }
    if (threadIdx.x == 0 && sub == 0) XB_TRACE(4);
    cluster_sync_all(); // every partial of this sub-tile is in place
    if (threadIdx.x == 0 && sub == 0) XB_TRACE(5);
    const int row0 = m0 + sub * TC_BM; // local output index of row 0 of the sub-tile
    if (nsplit <= 4)
      reduce_columns<NW, 4>(fo, red, red_s, row0, M, c_lo, c_hi, my_split, nsplit, map, st,
                            live, flags);
    else
      reduce_columns<NW, 8>(fo, red, red_s, row0, M, c_lo, c_hi, my_split, nsplit, map, st,
                            live, flags);
    cluster_sync_all(); // the partials are read before the next sub-tile overwrites them
  }
}

// A_MN = false: A = W tile [NSUB*128 rows][32 K] (forward, K-major; one TMA box)
// A_MN = true : A = W^T tile, i.e. W[32 K-rows][NSUB*128 columns] (backward,
//               MN-major): 4*NSUB 32x32 TMA boxes (128B/32B-atom swizzle) per
//               stage, one per 32-column MN atom, 4 KB apart
// X3 = true   : 3xTF32.  Warps 2-7 split every landed stage in place into hi
//               and a lo copy (generic-proxy writes, then fence.proxy.async);
//               the MMA thread issues hi*hi + hi*lo + lo*hi per K-step, which
//               recovers ~fp32 accuracy of the products at 3x the tensor work.
//               Warps 4-7 run the epilogue (TMEM lane quarter = warp % 4).
// B operand   : pass 0 streams the slab's x~ rows with one bn-row box (tm_b);
//               a re-issue pass streams ceil(n/32) 32-row boxes of the
//               compacted rows (tm_r), the MMA N is round_up(n, 16).
// FUSED + fo.loop: bound management runs inside the launch.  After a pass,
//               a grid barrier; every CTA compacts the pass's saturation
//               flags (same ascending order everywhere), prepares its share of
//               the re-issued x~ rows (DAC at m + 1, fp64), a second grid
//               barrier, and the next pass streams W again (L2-resident when
//               it fits).  The host never waits on the device.
template <bool A_MN, bool X3, int NSUB, bool FUSED>
__global__ void __launch_bounds__(tc_threads<X3, FUSED>(), 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                   const __grid_constant__ CUtensorMap tm_r,
                   const __grid_constant__ CUtensorMap tm_1, int M, int K, int B, int bn,
                   int kblocks_per_split, float *__restrict__ part, int ldp, size_t split_stride,
                   const int *__restrict__ n_rows, const __grid_constant__ FusedOut fo) {
  constexpr int STAGES = tc_stages<X3, NSUB>();
  constexpr int SB = tc_stage_bytes<X3, NSUB>();
  constexpr int AB = NSUB * TC_A_BYTES;          // A bytes per stage
  constexpr int LO = NSUB * TC_A_BYTES + TC_B_BYTES; // offset of the lo copies (X3)
  constexpr int NT = tc_threads<X3, FUSED>();
  static_assert(!FUSED || NT == XB_PREP_THREADS, "the in-kernel x~ prep shares prep_row's layout");
  extern __shared__ uint8_t smem_raw[];
  __shared__ float red[40];
  // 1024-byte alignment for the 128-byte swizzle atoms; stage s holds
  // [A | B | A_lo | B_lo]
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t *bars = (uint64_t *)(smem + STAGES * SB);
  uint32_t *tmem_slot = (uint32_t *)(bars + 3 * STAGES + 1);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + STAGES),
                 conv0 = smem_u32(bars + 2 * STAGES), done = smem_u32(bars + 3 * STAGES);
  auto stage_a = [&](int s) { return smem + s * SB; };
  auto stage_b = [&](int s) { return smem + s * SB + AB; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) XB_TRACE(0);
  const int m0 = blockIdx.x * TC_BM * NSUB;
  const int split = blockIdx.y;
  const int kb0 = split * kblocks_per_split;
  const int nkb = min(kblocks_per_split, (K + TC_BK - 1) / TC_BK - kb0);
  constexpr int CONV_THREADS = NT - 64;
  constexpr uint32_t TMEM_COLS = NSUB * TC_MAX_BN; // 256 or all 512 columns

  // rows (samples) of the first pass: pass 0 = the whole slab; a host-driven
  // re-issue (FUSED with fo.n_dev, or unfused with n_rows) = the compacted count
  const int *ndev = FUSED ? fo.n_dev : n_rows;
  int n = ndev ? *ndev : B;
  if (n <= 0) return; // nothing saturated: the whole grid leaves before any setup

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_b)) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
      mbar_init(conv0 + 8 * s, CONV_THREADS);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) { // TMEM: NSUB accumulators of 256 fp32 columns x 128 lanes
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  const int *map = FUSED ? fo.bm.map : nullptr; // compacted list (re-issue passes)
  bool reissue = ndev != nullptr;               // B operand = compacted rows (tm_r)
  bool level1 = false; // B operand = the prestaged m = 1 slab (tm_1), all columns
  int pass = FUSED ? fo.pass : 0;
  uint32_t gk = 0;     // k-blocks streamed by this CTA in this launch (ring position)
  uint32_t iter = 0;   // passes run in this launch (parity of `done`)
  unsigned bar_target = 0;
  const unsigned nctas = gridDim.x * gridDim.y;

  for (;;) {
    const int bnr = reissue ? max(16, (n + 15) / 16 * 16) : bn; // MMA N of this pass
    // a re-issue of a few samples streams just their x~ rows (32-row boxes);
    // of many, the slab's whole box (rows >= n are stale and never read out)
    const bool boxes = reissue && n <= 64;
    const int ncols = level1 ? fo.nb : n; // output columns of this pass
    const int nbox = (n + 31) / 32;
    const uint32_t b_bytes = boxes ? (uint32_t)nbox * 32u * TC_BK * 4u : (uint32_t)bn * TC_BK * 4;
    if (warp == 0 && lane == 0 && nkb > 0) {
      // ---------------- TMA producer
      // Pass 0 is launched as a programmatic dependent of the prep kernel: the
      // W tiles of the first stages stream while prep finishes; the x~ tiles
      // wait for it (griddepcontrol.wait).  Every later stage waits for a
      // free slot, i.e. after the first ones were consumed.
      const int pre = iter == 0 ? min(nkb, STAGES) : 0;
      auto load_a = [&](int kb, int s) {
        const int kk = (kb0 + kb) * TC_BK;
        if (A_MN) {
#pragma unroll
          for (int a = 0; a < NSUB * TC_BM / 32; ++a)
            tma_load_2d(smem_u32(stage_a(s) + a * 4096), &tm_a, full0 + 8 * s, m0 + 32 * a, kk);
        } else {
          tma_load_2d(smem_u32(stage_a(s)), &tm_a, full0 + 8 * s, kk, m0);
        }
      };
      for (int kb = 0; kb < pre; ++kb) { // fresh ring: slots kb are free
        mbar_expect_tx(full0 + 8 * kb, AB + b_bytes);
        load_a(kb, kb);
      }
      if (iter == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
      for (int kb = 0; kb < nkb; ++kb) {
        const uint32_t g = gk + (uint32_t)kb;
        const int s = (int)(g % STAGES);
        const uint32_t ph = (g / STAGES) & 1u;
        const int kk = (kb0 + kb) * TC_BK;
        if (kb >= pre) {
          mbar_wait(empty0 + 8 * s, ph ^ 1u);
          mbar_expect_tx(full0 + 8 * s, AB + b_bytes);
          load_a(kb, s);
        }
        if (boxes) {
          for (int j = 0; j < nbox; ++j)
            tma_load_2d(smem_u32(stage_b(s) + j * 4096), &tm_r, full0 + 8 * s, kk, 32 * j);
        } else if (level1) {
          tma_load_2d(smem_u32(stage_b(s)), &tm_1, full0 + 8 * s, kk, 0);
        } else {
          tma_load_2d(smem_u32(stage_b(s)), &tm_b, full0 + 8 * s, kk, 0);
        }
      }
    } else if (warp == 1 && lane == 0 && nkb > 0) {
      // ---------------- MMA issuer (one thread)
      const uint32_t idesc = idesc_tf32(bnr, A_MN);
      const uint32_t a_lbo = A_MN ? 4096u : 16u, a_sbo = A_MN ? 512u : 1024u;
      const uint32_t a_layout = A_MN ? 1u : 2u;
      // one MMA = 8 tf32 of K: K-major advances 32 bytes (+2 in 16-byte units),
      // MN-major advances 8 K-rows = two 4-row groups (+1024 bytes = +64)
      const uint32_t a_step = A_MN ? 64u : 2u;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int kb = 0; kb < nkb; ++kb) {
        const uint32_t g = gk + (uint32_t)kb;
        const int s = (int)(g % STAGES);
        const uint32_t ph = (g / STAGES) & 1u;
        mbar_wait((X3 ? conv0 : full0) + 8 * s, ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (kb == 0 && iter == 0) XB_TRACE(1);
        if (kb == 0 && iter == 1) XB_TRACE(11);
        const uint64_t db = umma_desc(smem_u32(stage_b(s)), 16u, 1024u, 2u);
        const uint64_t dbl = umma_desc(smem_u32(stage_b(s) + LO), 16u, 1024u, 2u);
#pragma unroll
        for (int sub = 0; sub < NSUB; ++sub) {
          // sub-tile: K-major rows 128*sub.. (16 KB further); MN-major atoms 4*sub..
          const uint64_t da =
              umma_desc(smem_u32(stage_a(s) + sub * TC_A_BYTES), a_lbo, a_sbo, a_layout);
          const uint64_t dal =
              umma_desc(smem_u32(stage_a(s) + LO + sub * TC_A_BYTES), a_lbo, a_sbo, a_layout);
          const uint32_t acc = tmem + (uint32_t)(sub * TC_MAX_BN);
#pragma unroll
          for (int k = 0; k < TC_BK / 8; ++k) {
            mma_tf32(acc, da + a_step * k, db + 2u * k, idesc, (kb | k) != 0);
            if (X3) {
              mma_tf32(acc, da + a_step * k, dbl + 2u * k, idesc, 1u);
              mma_tf32(acc, dal + a_step * k, db + 2u * k, idesc, 1u);
            }
          }
        }
        mma_commit(empty0 + 8 * s); // smem stage free once these MMAs retire
      }
      mma_commit(done);
    } else if (X3 && warp >= 2 && nkb > 0) {
      // ---------------- hi/lo split of each landed stage (3xTF32)
      const int ct = threadIdx.x - 64;
      const int n4 = (AB + (int)b_bytes) / 16; // B follows A directly in both halves
      for (int kb = 0; kb < nkb; ++kb) {
        const uint32_t g = gk + (uint32_t)kb;
        const int s = (int)(g % STAGES);
        const uint32_t ph = (g / STAGES) & 1u;
        mbar_wait(full0 + 8 * s, ph);
        float4 *a4 = reinterpret_cast<float4 *>(stage_a(s));
        float4 *al4 = reinterpret_cast<float4 *>(stage_a(s) + LO);
        for (int e = ct; e < n4; e += CONV_THREADS) {
          float4 v = a4[e], lo;
          split_tf32(v, lo);
          a4[e] = v;
          al4[e] = lo;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(conv0 + 8 * s) : "memory");
      }
    }
    __syncwarp();
    if (iter == 0) asm volatile("griddepcontrol.wait;" ::: "memory"); // prep's st[] / flags
    if (FUSED && !X3 && iter == 0 && fo.loop && fo.xt1 && warp >= 2) stage_level1(fo, red);

    // ---------------- epilogue: TMEM -> registers -> partial sums / output stage
    if (nkb > 0) {
      mbar_wait(done, iter & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (threadIdx.x == 0 && iter == 0) XB_TRACE(2);
      if (threadIdx.x == 0 && iter == 1) XB_TRACE(12);
    }
    const int quarter = warp & 3;
    if (!FUSED) {
      constexpr int EPI_W0 = X3 ? 4 : 0;
      if (warp >= EPI_W0 && warp < EPI_W0 + 4) {
        float *dst = part + (size_t)split * split_stride;
#pragma unroll
        for (int sub = 0; sub < NSUB; ++sub) {
          const int o = m0 + sub * TC_BM + quarter * 32 + lane;
          for (int c0 = 0; c0 < bnr; c0 += 32) {
            uint32_t r[32];
            XB_TMEM_LD32(tmem + ((uint32_t)(quarter * 32) << 16) +
                             (uint32_t)(sub * TC_MAX_BN + c0),
                         r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (o < M) {
#pragma unroll
              for (int c = 0; c < 32; ++c) {
                const int b = c0 + c;
                if (b < n) dst[(size_t)b * ldp + o] = nkb > 0 ? __uint_as_float(r[c]) : 0.f;
              }
            }
          }
        }
      }
      break;
    }
    // split peers: cluster (1, S), CTA rank == split index
    fused_output_stage<NT / 32, NSUB>(fo, tmem, smem, nkb, m0, M, ncols, bnr, cluster_rank(),
                                      cluster_size(), reissue ? map : nullptr, pass, level1);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    gk += (uint32_t)max(nkb, 0);
    ++iter;
    if (!fo.loop) break;
    // ---------------- in-kernel bound management: next re-issue pass
    bar_target += nctas;
    grid_sync(fo.bar, bar_target); // every flag of this pass is final
    if (threadIdx.x == 0 && iter == 1) XB_TRACE(8);
    const int nb = fo.nb;
    n = block_compact(fo.bm.flags + (pass & 1) * nb, nb, fo.n0, fo.bm.map,
                      reinterpret_cast<int *>(red));
#ifdef XB_TC_TRACE
    if (threadIdx.x == 0 && iter == 1 && blockIdx.x + gridDim.x * blockIdx.y < 4096)
      g_tc_trace[blockIdx.x + gridDim.x * blockIdx.y][15] = (unsigned long long)n;
#endif
    if (n == 0) break; // uniform: every CTA read the same flags
    if (pass == 0 && fo.xt1) {
      // first re-issue from the prestaged m = 1 slab: nothing to prepare, and
      // the flags pass 1 writes are still clear from the prep kernel -- so no
      // second barrier either
      level1 = true;
      ++pass;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      continue;
    }
    {
      // clear the flags the next pass will write (read by nobody now)
      int *nf = fo.bm.flags + ((pass + 1) & 1) * nb;
      const unsigned cta = blockIdx.x + gridDim.x * blockIdx.y;
      for (int i = (int)(cta * NT) + threadIdx.x; i < nb; i += (int)(nctas * NT)) nf[i] = 0;
      // this CTA's share of the re-issued rows: x~ at m + 1 (io.cpp:117-131)
      for (int c = (int)cta; c < n; c += (int)nctas) {
        const int b = fo.bm.map[c];
        SampleState s = level1 ? fo.st1[b] : fo.st[b]; // its state in the pass just run
        s.m += 1;
        s.norm = prep_row(fo.X + (size_t)b * fo.K, fo.K, fo.xt + (size_t)c * fo.ldt, s, fo.io,
                          fo.key, fo.seq0 + (uint64_t)b, fo.in0, red);
        if (threadIdx.x == 0) fo.st[b] = s;
      }
      if (threadIdx.x == 0 && iter == 1) XB_TRACE(14);
      // the x~ rows are read by other CTAs' TMA (async proxy)
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    if (threadIdx.x == 0 && iter == 1) XB_TRACE(9);
    bar_target += nctas;
    grid_sync(fo.bar, bar_target);
    if (threadIdx.x == 0 && iter == 1) XB_TRACE(10);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    reissue = true;
    level1 = false;
    ++pass;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) XB_TRACE(3);
#ifdef XB_TC_TRACE
  if (threadIdx.x == 0 && blockIdx.x + gridDim.x * blockIdx.y < 4096)
    g_tc_trace[blockIdx.x + gridDim.x * blockIdx.y][7] = iter;
  if (threadIdx.x == 0 && blockIdx.x + gridDim.x * blockIdx.y < 4096)
    g_tc_trace[blockIdx.x + gridDim.x * blockIdx.y][13] = (unsigned long long)n;
#endif
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS));
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  });
  if (!fn) raise("cuTensorMapEncodeTiled unavailable (driver too old for TMA)");
  return fn;
}

// 2-D fp32 tensor map over a row-major [rows][cols] array with row stride ld
// floats; box = [box_rows][32 floats], 128-byte swizzle (16- or 32-byte
// granule), OOB zero fill
CUtensorMap encode_map(const float *base, int rows, int cols, int ld, int box_rows,
                       CUtensorMapSwizzle swz) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  const cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)base, dims, strides,
                           box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) raise("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

// A launch needs up to four maps and a call re-uses the same tile and
// scratch buffers, so the encodings (a driver call each) are kept in a small
// per-thread cache keyed by every argument: a hit is the same 128-byte map.
CUtensorMap make_map(const float *base, int rows, int cols, int ld, int box_rows,
                     CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  struct Entry {
    const float *base;
    int rows, cols, ld, box;
    CUtensorMapSwizzle swz;
    CUtensorMap map;
  };
  constexpr int N = 16;
  thread_local Entry cache[N];
  thread_local int used = 0, next = 0;
  for (int i = 0; i < used; ++i) {
    const Entry &e = cache[i];
    if (e.base == base && e.rows == rows && e.cols == cols && e.ld == ld && e.box == box_rows &&
        e.swz == swz)
      return e.map;
  }
  Entry &e = cache[next];
  e.map = encode_map(base, rows, cols, ld, box_rows, swz);
  e.base = base;
  e.rows = rows;
  e.cols = cols;
  e.ld = ld;
  e.box = box_rows;
  e.swz = swz;
  next = (next + 1) % N;
  used = used < N ? used + 1 : N;
  return e.map;
}

} // namespace

// 128-row sub-tiles per CTA.  Two halve the x~ re-reads but need twice the
// K-splits to fill the SMs (more partial-sum traffic): measured on B200 they
// win for 16384^2 (forward 571 vs 607 us, backward 263 vs 278 us) and lose
// for 4096^2 (70 vs 66 us); one for 3xTF32 (its stage would not fit twice)
// (fused output stage, round 1: NSUB = 2 at 4096^2 doubles the forward,
// 71 vs 36 us back to back; at 16384^2 the two are equal, 265 us)
#ifndef XB_TC_NSUB2_MIN
#define XB_TC_NSUB2_MIN 8192
#endif
static int tc_nsub(int M, bool x3) { return (!x3 && M >= XB_TC_NSUB2_MIN) ? 2 : 1; }

int tc_splits(int M, int K, bool x3) {
  const int band = TC_BM * tc_nsub(M, x3);
  const int mt = (M + band - 1) / band;
  const int kbs = (K + TC_BK - 1) / TC_BK;
  int s = std::max(1, 148 / std::max(mt, 1));
  s = std::min(s, std::max(1, kbs / 4)); // keep >= 4 K-blocks per split
  return std::max(1, std::min(s, 16));
}

struct TcArgs {
  dim3 grid;
  cudaStream_t st;
  CUtensorMap ma, mb, mr, m1;
  int M, K, nb, bn, per;
  float *part;
  size_t split_stride;
  const int *n_rows;
  FusedOut fo;
  bool pdl; // programmatic dependent of the preceding kernel
};

// launch one contraction; check_loop: only report whether every cluster of
// the grid can be resident at once (the in-kernel BM loop needs it)
template <bool A_MN, bool X3, int NSUB, bool FUSED>
static bool launch_tc(const TcArgs &a, bool check_loop) {
  auto kern = tc_gemm_kernel<A_MN, X3, NSUB, FUSED>;
  static std::atomic<uint64_t> configured{0};
  once_per_device(configured, [&] {
    XB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 tc_smem<X3, NSUB>()));
    if (FUSED) XB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
  });
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = a.grid;
  cfg.blockDim = dim3(tc_threads<X3, FUSED>());
  cfg.dynamicSmemBytes = tc_smem<X3, NSUB>();
  cfg.stream = a.st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (FUSED) { // the K-splits of one M-tile form one cluster
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 1;
    attr[na].val.clusterDim.y = a.grid.y;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (a.pdl) { // pass 0: may start while the prep kernel finishes (griddepcontrol)
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  if (check_loop) {
    int clusters = 0;
    if (!FUSED || cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return clusters >= (int)a.grid.x;
  }
  XB_CUDA(cudaLaunchKernelEx(&cfg, kern, a.ma, a.mb, a.mr, a.m1, a.M, a.K, a.nb, a.bn, a.per, a.part,
                             a.M, a.split_stride, a.n_rows, a.fo));
  count_launch();
  XB_CUDA(cudaGetLastError());
  return true;
}

template <bool FUSED>
static bool launch_variant(bool transposed, bool x3, int nsub, const TcArgs &a, bool check) {
  if (x3)
    return transposed ? launch_tc<true, true, 1, FUSED>(a, check)
                      : launch_tc<false, true, 1, FUSED>(a, check);
  if (nsub == 2)
    return transposed ? launch_tc<true, false, 2, FUSED>(a, check)
                      : launch_tc<false, false, 2, FUSED>(a, check);
  return transposed ? launch_tc<true, false, 1, FUSED>(a, check)
                    : launch_tc<false, false, 1, FUSED>(a, check);
}

// XB_NO_PDL=1: launch pass 0 in plain stream order (A/B measurements)
static bool pdl_disabled() {
  const char *e = getenv("XB_NO_PDL");
  return e && e[0] == '1';
}

// contraction on tcgen05.
//   forward : o = row of W, K = columns of W   (A = W, K-major)
//   backward: o = column of W, K = rows of W   (A = W^T, MN-major)
// fo == nullptr: partial sums part[s][b][o] (split stride B x M) for the
// epilogue kernel; n_dev != nullptr: a compacted re-issue whose row count is
// on the device.  Otherwise the cluster-fused output stage writes fo->Y, per
// N slab of <= 256 samples (fo->bm points at slab 0's buffers; slab k uses
// flags + 512 k, counts + 64 k, map + 256 k, bar + k).  bm_loop: every BM
// re-issue runs inside the launch; false when the grid could not be
// co-resident (the caller then drives the re-issue passes).
bool tc_gemm(Tile &t, bool transposed, bool x3, const float *Xt, int ldt, int B, float *part,
             int splits, const FusedOut *fo, const int *n_dev, bool bm_loop) {
  const int M = transposed ? t.C : t.R, K = transposed ? t.R : t.C;
  const int nsub = tc_nsub(M, x3);
  const int kbs = (K + TC_BK - 1) / TC_BK;
  const int per = (kbs + splits - 1) / splits;
  const int used = (kbs + per - 1) / per;
  bool looped = bm_loop;
  for (int n0 = 0; n0 < B; n0 += TC_MAX_BN) {
    const int nb = std::min(TC_MAX_BN, B - n0);
    const int bn = std::max(16, (nb + 15) / 16 * 16);
    TcArgs a;
    // W as [R][C] with row stride ld: the forward box is 128*nsub rows x 32
    // columns, the backward box 32 rows (K) x 32 columns (one MN atom)
    a.ma = transposed ? make_map(t.W, t.R, t.C, t.ld, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)
                      : make_map(t.W, t.R, t.C, t.ld, TC_BM * nsub);
    a.mb = make_map(Xt + (size_t)n0 * ldt, nb, K, ldt, bn);
    a.mr = make_map(Xt + (size_t)n0 * ldt, nb, K, ldt, 32);
    a.m1 = (fo && fo->xt1) ? make_map(fo->xt1 + (size_t)n0 * ldt, nb, K, ldt, bn) : a.mb;
    a.grid = dim3((M + TC_BM * nsub - 1) / (TC_BM * nsub), used);
    a.st = t.stream;
    a.M = M;
    a.K = K;
    a.nb = nb;
    a.bn = bn;
    a.per = per;
    a.n_rows = n_dev;
    a.pdl = !n_dev && !(fo && fo->n_dev) && !pdl_disabled();
    if (fo) {
      a.fo = *fo;
      const int slab = n0 / TC_MAX_BN;
      a.fo.n0 = fo->n0 + n0; // global index of the slab's first sample
      a.fo.nb = nb;
      a.fo.bm.flags = fo->bm.flags + (size_t)BM_SLAB_WORDS * slab;
      a.fo.bm.counts = fo->bm.counts + (size_t)BM_SLAB_WORDS * slab;
      a.fo.bm.map = fo->bm.map + n0;
      a.fo.bar = fo->bar ? fo->bar + slab : nullptr;
      a.fo.xt = fo->xt ? fo->xt + (size_t)n0 * ldt : nullptr;
      a.fo.xt1 = fo->xt1 ? fo->xt1 + (size_t)n0 * ldt : nullptr;
      a.part = nullptr;
      a.split_stride = 0;
      if (bm_loop && n0 == 0) looped = launch_variant<true>(transposed, x3, nsub, a, true);
      a.fo.loop = looped ? 1 : 0;
      launch_variant<true>(transposed, x3, nsub, a, false);
    } else {
      // partial sums of this N slab land at part + n0 rows, split stride B x M
      a.part = part + (size_t)n0 * M;
      a.split_stride = (size_t)B * M;
      a.fo = FusedOut{};
      launch_variant<false>(transposed, x3, nsub, a, false);
    }
  }
  return looped;
}

int tc_used_splits(int K, int splits) {
  const int kbs = (K + TC_BK - 1) / TC_BK;
  const int per = (kbs + splits - 1) / splits;
  return (kbs + per - 1) / per;
}

} // namespace xb
