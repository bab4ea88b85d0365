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
__device__ unsigned long long g_tc_trace[4096][4];
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
  return (int)cudaMemcpyFromSymbol(out, g_tc_trace, sizeof(unsigned long long) * 4 *
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
__device__ __forceinline__ float4 dsmem_ld4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
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

// Cluster-fused output stage.  Every warp of the CTA: drain this CTA's
// accumulator (NSUB sub-tiles of 128 TMEM lanes x bn columns) into its idle
// pipeline memory as [bn][128] fp32, cluster barrier, then reduce this CTA's
// share of the columns (samples) over the S split partials -- split r lives
// in cluster CTA peer0 + r * pstride -- through distributed shared memory
// (all S loads in flight, summed in split order like the epilogue kernel) and
// run the output stage (xb_mvm_common.cuh) straight into Y.
template <int NW, int NSUB>
__device__ __forceinline__ void fused_output_stage(const FusedOut &fo, uint32_t tmem,
                                                   uint8_t *smem, int nkb, int m0, int M, int B,
                                                   int bn, uint32_t my_split, uint32_t nsplit,
                                                   uint32_t peer0, uint32_t pstride) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, quarter = warp & 3;
  float *red = reinterpret_cast<float *>(smem);
  const uint32_t red_s = smem_u32(red);
  const int cols = (bn + (int)nsplit - 1) / (int)nsplit;
  const int c_lo = (int)my_split * cols, c_hi = min(bn, c_lo + cols);
#pragma unroll 1
  for (int sub = 0; sub < NSUB; ++sub) {
    const int row = quarter * 32 + lane;
    for (int c0 = 32 * (warp >> 2); c0 < bn; c0 += 32 * (NW / 4)) {
      uint32_t r[32];
      XB_TMEM_LD32(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(sub * TC_MAX_BN + c0), r);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int c = 0; c < 32; ++c) red[(c0 + c) * TC_BM + row] = nkb > 0 ? __uint_as_float(r[c]) : 0.f;
    }
    cluster_sync_all(); // every partial of this sub-tile is in place
    {
      // thread: group of 4 rows (grp) x every NW-th column of this CTA's range
      const int grp = threadIdx.x & 31, cph = threadIdx.x >> 5;
      const int row0 = m0 + sub * TC_BM; // local output index of row 0 of the sub-tile
      for (int c = c_lo + cph; c < c_hi; c += NW) {
        if (c >= B) break;
        const int b = fo.map ? fo.map[fo.n0 + c] : fo.n0 + c;
        const SampleState sst = fo.st[b];
        if (!fo.first_pass && !sst.active) continue;
        const uint32_t off = red_s + (uint32_t)((c * TC_BM + 4 * grp) * 4);
        float4 v[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) // all remote loads in flight, then the sum
          if (r < (int)nsplit) v[r] = dsmem_ld4(dsmem_map(off, peer0 + (uint32_t)r * pstride));
        float4 acc4 = v[0];
#pragma unroll
        for (int r = 1; r < 8; ++r) // split order (as the epilogue kernel)
          if (r < (int)nsplit) {
            acc4.x += v[r].x;
            acc4.y += v[r].y;
            acc4.z += v[r].z;
            acc4.w += v[r].w;
          }
        if (row0 + 4 * grp >= M) continue;
        const float a[4] = {acc4.x, acc4.y, acc4.z, acc4.w};
        // global output index of this group: o0 + row0 + 4 grp (o0 % 4 == 0 on
        // the fused path, so groups align with the noise groups)
        const int g = (fo.o0 + row0) / 4 + grp;
        const bool hit = epilogue_group4(a, g, fo.o0, M, sst, fo.io, fo.key,
                                         fo.seq0 + (uint64_t)b, fo.Y + (size_t)b * fo.ldy);
        bm_flag(hit, sst, fo.io, fo.sat, b, fo.B, fo.pass_slot);
      }
    }
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
template <bool A_MN, bool X3, int NSUB, bool FUSED>
__global__ void __launch_bounds__(tc_threads<X3, FUSED>(), 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                   int M, int K, int B, int bn, int kblocks_per_split, float *__restrict__ part,
                   int ldp, size_t split_stride, const __grid_constant__ FusedOut fo) {
  constexpr int STAGES = tc_stages<X3, NSUB>();
  constexpr int SB = tc_stage_bytes<X3, NSUB>();
  constexpr int AB = NSUB * TC_A_BYTES;          // A bytes per stage
  constexpr int LO = NSUB * TC_A_BYTES + TC_B_BYTES; // offset of the lo copies (X3)
  extern __shared__ uint8_t smem_raw[];
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
  constexpr int CONV_THREADS = tc_threads<X3, FUSED>() - 64;
  constexpr uint32_t TMEM_COLS = NSUB * TC_MAX_BN; // 256 or all 512 columns

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
  const uint32_t b_bytes = (uint32_t)bn * TC_BK * 4;

  if (warp == 0 && lane == 0 && nkb > 0) {
    // ---------------- TMA producer
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (uint32_t)(kb / STAGES) & 1u;
      mbar_wait(empty0 + 8 * s, ph ^ 1u);
      mbar_expect_tx(full0 + 8 * s, AB + b_bytes);
      const int kk = (kb0 + kb) * TC_BK;
      if (A_MN) {
#pragma unroll
        for (int a = 0; a < NSUB * TC_BM / 32; ++a)
          tma_load_2d(smem_u32(stage_a(s) + a * 4096), &tm_a, full0 + 8 * s, m0 + 32 * a, kk);
      } else {
        tma_load_2d(smem_u32(stage_a(s)), &tm_a, full0 + 8 * s, kk, m0);
      }
      tma_load_2d(smem_u32(stage_b(s)), &tm_b, full0 + 8 * s, kk, 0);
    }
  } else if (warp == 1 && lane == 0 && nkb > 0) {
    // ---------------- MMA issuer (one thread)
    const uint32_t idesc = idesc_tf32(bn, A_MN);
    const uint32_t a_lbo = A_MN ? 4096u : 16u, a_sbo = A_MN ? 512u : 1024u;
    const uint32_t a_layout = A_MN ? 1u : 2u;
    // one MMA = 8 tf32 of K: K-major advances 32 bytes (+2 in 16-byte units),
    // MN-major advances 8 K-rows = two 4-row groups (+1024 bytes = +64)
    const uint32_t a_step = A_MN ? 64u : 2u;
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (uint32_t)(kb / STAGES) & 1u;
      mbar_wait((X3 ? conv0 : full0) + 8 * s, ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (kb == 0) XB_TRACE(1);
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
      const int s = kb % STAGES;
      const uint32_t ph = (uint32_t)(kb / STAGES) & 1u;
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

  // ---------------- epilogue: TMEM -> registers -> partial sums
  constexpr int EPI_W0 = X3 ? 4 : 0;
  const bool epi_warp = warp >= EPI_W0 && warp < EPI_W0 + 4;
  if (epi_warp && nkb > 0) {
    mbar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x == 32 * EPI_W0) XB_TRACE(2);
  }
  const int quarter = warp & 3;
  if (!FUSED) {
    if (epi_warp) {
      float *dst = part + (size_t)split * split_stride;
#pragma unroll
      for (int sub = 0; sub < NSUB; ++sub) {
        const int o = m0 + sub * TC_BM + quarter * 32 + lane;
        for (int c0 = 0; c0 < bn; c0 += 32) {
          uint32_t r[32];
          XB_TMEM_LD32(tmem + ((uint32_t)(quarter * 32) << 16) +
                           (uint32_t)(sub * TC_MAX_BN + c0),
                       r);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (o < M) {
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              const int b = c0 + c;
              if (b < B) dst[(size_t)b * ldp + o] = nkb > 0 ? __uint_as_float(r[c]) : 0.f;
            }
          }
        }
      }
    }
  } else {
    if (!epi_warp && nkb > 0) {
      mbar_wait(done, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    // split peers: cluster (1, S), CTA rank == split index
    fused_output_stage<tc_threads<X3, FUSED>() / 32, NSUB>(fo, tmem, smem, nkb, m0, M, B, bn,
                                                            cluster_rank(), cluster_size(), 0u,
                                                            1u);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) XB_TRACE(3);
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS));
}

// ============================================================ CTA pairs
// 2-SM variant (cta_group::2).  A cluster (2, S): the two CTAs of a pair own
// consecutive 128-row M-tiles of one K-split; each streams its own A tile and
// HALF of the x~ tile (bn/2 samples) -- signalling the leader's full barrier
// through the 2-SM TMA form -- and the leader issues M=256 UMMAs that read A
// and B from both CTAs' shared memory, each CTA accumulating its 128 rows in
// its own TMEM.  Per stage a CTA holds 16 + 16 KB instead of 16 + 32 KB: six
// stages in flight instead of four, and half the x~ re-reads from L2.
constexpr int TP_STAGES = 6;
constexpr int TP_STAGE = TC_A_BYTES + TC_B_BYTES / 2; // 32 KB
constexpr int TP_SMEM = TP_STAGES * TP_STAGE + 1024 + 256;

__device__ __forceinline__ uint32_t cluster_ctaid_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctaid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_ctaid_y() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctaid.y;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_nctaid_y() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctaid.y;" : "=r"(r));
  return r;
}
// arrive (+ expected bytes) on an mbarrier of another CTA of the cluster
__device__ __forceinline__ void mbar_expect_tx_cluster(uint32_t cbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(
                   cbar),
               "r"(bytes)
               : "memory");
}
// TMA into this CTA's shared memory, completion counted on the pair leader's
// mbarrier (cbar: shared::cluster address)
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap *map,
                                                 uint32_t cbar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(cbar)
      : "memory");
}
__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_d, uint64_t a, uint64_t b,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
// arrive on the same mbarrier offset in both CTAs of the pair (mask: cluster ranks)
__device__ __forceinline__ void mma_commit_pair(uint32_t bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::"
               "cluster.b64 [%0], %1;" ::"r"(bar),
               "h"(mask)
               : "memory");
}

template <bool A_MN, bool FUSED>
__global__ void __launch_bounds__(tc_threads<false, FUSED>(), 1)
    tc_pair_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                   int M, int K, int B, int bn, int kblocks_per_split, float *__restrict__ part,
                   int ldp, size_t split_stride, const __grid_constant__ FusedOut fo) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t *bars = (uint64_t *)(smem + TP_STAGES * TP_STAGE);
  uint32_t *tmem_slot = (uint32_t *)(bars + 2 * TP_STAGES + 1);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + TP_STAGES),
                 done = smem_u32(bars + 2 * TP_STAGES);
  auto stage_a = [&](int s) { return smem + s * TP_STAGE; };
  auto stage_b = [&](int s) { return smem + s * TP_STAGE + TC_A_BYTES; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t xr = cluster_ctaid_x();      // 0 = pair leader (issues the MMAs), 1 = peer
  const uint32_t my_rank = cluster_rank();
  const uint32_t lead_rank = my_rank - xr;    // ranks: x + 2 y
  const uint16_t pair_mask = (uint16_t)(3u << lead_rank);
  const int m0 = blockIdx.x * TC_BM;
  const int split = blockIdx.y;
  const int kb0 = split * kblocks_per_split;
  const int nkb = min(kblocks_per_split, (K + TC_BK - 1) / TC_BK - kb0);
  const int half = bn / 2;

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_b)) : "memory");
    for (int s = 0; s < TP_STAGES; ++s) {
      mbar_init(full0 + 8 * s, 2); // both producers of the pair arrive on the leader's
      mbar_init(empty0 + 8 * s, 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) { // TMEM, allocated by the pair together
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TC_MAX_BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all(); // barriers of both CTAs initialised, TMEM allocated
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t bytes_per_cta = TC_A_BYTES + (uint32_t)half * TC_BK * 4;
  const uint32_t lead_full0 = dsmem_map(full0, lead_rank);

  if (warp == 0 && lane == 0 && nkb > 0) {
    // ---------------- TMA producer (both CTAs)
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % TP_STAGES;
      const uint32_t ph = (uint32_t)(kb / TP_STAGES) & 1u;
      mbar_wait(empty0 + 8 * s, ph ^ 1u);
      mbar_expect_tx_cluster(lead_full0 + 8 * s, bytes_per_cta);
      const int kk = (kb0 + kb) * TC_BK;
      if (A_MN) {
#pragma unroll
        for (int a = 0; a < TC_BM / 32; ++a)
          tma_load_2d_pair(smem_u32(stage_a(s) + a * 4096), &tm_a, lead_full0 + 8 * s,
                           m0 + 32 * a, kk);
      } else {
        tma_load_2d_pair(smem_u32(stage_a(s)), &tm_a, lead_full0 + 8 * s, kk, m0);
      }
      tma_load_2d_pair(smem_u32(stage_b(s)), &tm_b, lead_full0 + 8 * s, kk, (int)xr * half);
    }
  } else if (warp == 1 && lane == 0 && xr == 0 && nkb > 0) {
    // ---------------- MMA issuer: the pair leader, M = 256 across both CTAs
    const uint32_t idesc =
        (idesc_tf32(bn, A_MN) & ~(0x1Fu << 24)) | ((uint32_t)(2 * TC_BM >> 4) << 24);
    const uint32_t a_lbo = A_MN ? 4096u : 16u, a_sbo = A_MN ? 512u : 1024u;
    const uint32_t a_layout = A_MN ? 1u : 2u;
    const uint32_t a_step = A_MN ? 64u : 2u;
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % TP_STAGES;
      const uint32_t ph = (uint32_t)(kb / TP_STAGES) & 1u;
      mbar_wait(full0 + 8 * s, ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint64_t da = umma_desc(smem_u32(stage_a(s)), a_lbo, a_sbo, a_layout);
      const uint64_t db = umma_desc(smem_u32(stage_b(s)), 16u, 1024u, 2u);
#pragma unroll
      for (int k = 0; k < TC_BK / 8; ++k)
        mma_tf32_pair(tmem, da + a_step * k, db + 2u * k, idesc, (kb | k) != 0);
      mma_commit_pair(empty0 + 8 * s, pair_mask); // both CTAs may refill stage s
    }
    mma_commit_pair(done, pair_mask);
  }
  __syncwarp();

  // ---------------- epilogue: each CTA drains its own 128 accumulator rows
  if (nkb > 0) {
    mbar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  if (!FUSED) {
    if (warp < 4) {
      const int o = m0 + warp * 32 + lane;
      float *dst = part + (size_t)split * split_stride;
      for (int c0 = 0; c0 < bn; c0 += 32) {
        uint32_t r[32];
        XB_TMEM_LD32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (o < M) {
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const int b = c0 + c;
            if (b < B) dst[(size_t)b * ldp + o] = nkb > 0 ? __uint_as_float(r[c]) : 0.f;
          }
        }
      }
    }
  } else {
    // split peers: cluster (2, S), rank = x + 2 y
    fused_output_stage<tc_threads<false, FUSED>() / 32, 1>(fo, tmem, smem, nkb, m0, M, B, bn,
                                                            cluster_ctaid_y(), cluster_nctaid_y(),
                                                            xr, 2u);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all(); // both CTAs are done with the pair's TMEM
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TC_MAX_BN));
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
CUtensorMap make_map(const float *base, int rows, int cols, int ld, int box_rows,
                     CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
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

template <bool A_MN, bool X3, int NSUB, bool FUSED>
static void launch_tc(dim3 grid, cudaStream_t st, const CUtensorMap &ma, const CUtensorMap &mb,
                      int M, int K, int nb, int bn, int per, float *part, size_t split_stride,
                      const FusedOut &fo) {
  auto kern = tc_gemm_kernel<A_MN, X3, NSUB, FUSED>;
  static std::atomic<uint64_t> configured{0};
  once_per_device(configured, [&] {
    XB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 tc_smem<X3, NSUB>()));
    if (FUSED) XB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
  });
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(tc_threads<X3, FUSED>());
  cfg.dynamicSmemBytes = tc_smem<X3, NSUB>();
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (FUSED) { // the K-splits of one M-tile form one cluster
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = grid.y;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  XB_CUDA(cudaLaunchKernelEx(&cfg, kern, ma, mb, M, K, nb, bn, per, part, M, split_stride, fo));
  count_launch();
  XB_CUDA(cudaGetLastError());
}

template <bool FUSED>
static void launch_variant(bool transposed, bool x3, int nsub, dim3 grid, cudaStream_t st,
                           const CUtensorMap &ma, const CUtensorMap &mb, int M, int K, int nb,
                           int bn, int per, float *p, size_t ss, const FusedOut &fo) {
  if (x3) {
    transposed ? launch_tc<true, true, 1, FUSED>(grid, st, ma, mb, M, K, nb, bn, per, p, ss, fo)
               : launch_tc<false, true, 1, FUSED>(grid, st, ma, mb, M, K, nb, bn, per, p, ss, fo);
  } else if (nsub == 2) {
    transposed ? launch_tc<true, false, 2, FUSED>(grid, st, ma, mb, M, K, nb, bn, per, p, ss, fo)
               : launch_tc<false, false, 2, FUSED>(grid, st, ma, mb, M, K, nb, bn, per, p, ss, fo);
  } else {
    transposed ? launch_tc<true, false, 1, FUSED>(grid, st, ma, mb, M, K, nb, bn, per, p, ss, fo)
               : launch_tc<false, false, 1, FUSED>(grid, st, ma, mb, M, K, nb, bn, per, p, ss, fo);
  }
}

template <bool A_MN, bool FUSED>
static void launch_pair(dim3 grid, cudaStream_t st, const CUtensorMap &ma, const CUtensorMap &mb,
                        int M, int K, int nb, int bn, int per, float *part, size_t split_stride,
                        const FusedOut &fo) {
  auto kern = tc_pair_kernel<A_MN, FUSED>;
  static std::atomic<uint64_t> configured{0};
  once_per_device(configured, [&] {
    XB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, TP_SMEM));
  });
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(tc_threads<false, FUSED>());
  cfg.dynamicSmemBytes = TP_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension; // (CTA pair) x (K-splits when fused)
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = FUSED ? grid.y : 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  XB_CUDA(cudaLaunchKernelEx(&cfg, kern, ma, mb, M, K, nb, bn, per, part, M, split_stride, fo));
  count_launch();
  XB_CUDA(cudaGetLastError());
}

// Opt-in (XB_TC_PAIR=1): correct (tests/test_gpu_mvm.py runs it) but measured
// slower on B200 for the bench shapes -- 4096^2 x 256 forward 109 us fused /
// 79 us unfused vs 62 / 65 us for the single-CTA kernel; tensor pipe 22 % --
// so the single-CTA kernel stays the default.
static bool pair_enabled() {
  const char *e = getenv("XB_TC_PAIR");
  return e && e[0] == '1';
}

// contraction on tcgen05.
//   forward : o = row of W, K = columns of W   (A = W, K-major)
//   backward: o = column of W, K = rows of W   (A = W^T, MN-major)
// fo == nullptr: partial sums part[s][b][o] (split stride B x M) for the
// epilogue kernel; otherwise the cluster-fused output stage writes fo->Y.
void tc_gemm(Tile &t, bool transposed, bool x3, const float *Xt, int ldt, int B, float *part,
             int splits, const FusedOut *fo) {
  const int M = transposed ? t.C : t.R, K = transposed ? t.R : t.C;
  const int nsub = tc_nsub(M, x3);
  const int kbs = (K + TC_BK - 1) / TC_BK;
  const int per = (kbs + splits - 1) / splits;
  const int used = (kbs + per - 1) / per;
  for (int n0 = 0; n0 < B; n0 += TC_MAX_BN) {
    const int nb = std::min(TC_MAX_BN, B - n0);
    const int bn = std::max(16, (nb + 15) / 16 * 16);
    // W as [R][C] with row stride ld: the forward box is 128*nsub rows x 32
    // columns, the backward box 32 rows (K) x 32 columns (one MN atom)
    const CUtensorMap ma =
        transposed ? make_map(t.W, t.R, t.C, t.ld, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)
                   : make_map(t.W, t.R, t.C, t.ld, TC_BM * nsub);
    const CUtensorMap mb = make_map(Xt + (size_t)n0 * ldt, nb, K, ldt, bn);
    const int mtiles = (M + TC_BM - 1) / TC_BM;
    const bool pair = !x3 && nsub == 1 && mtiles >= 2 && (!fo || used <= 4) && pair_enabled();
    if (pair) { // 2-SM UMMA: each CTA streams its A tile and half of the x~ tile
      const CUtensorMap mbh = make_map(Xt + (size_t)n0 * ldt, nb, K, ldt, bn / 2);
      const dim3 grid2((mtiles + 1) / 2 * 2, used);
      if (fo) {
        FusedOut f = *fo;
        f.n0 = n0;
        transposed ? launch_pair<true, true>(grid2, t.stream, ma, mbh, M, K, nb, bn, per, nullptr,
                                             0, f)
                   : launch_pair<false, true>(grid2, t.stream, ma, mbh, M, K, nb, bn, per,
                                              nullptr, 0, f);
      } else {
        float *p = part + (size_t)n0 * M;
        transposed ? launch_pair<true, false>(grid2, t.stream, ma, mbh, M, K, nb, bn, per, p,
                                              (size_t)B * M, FusedOut{})
                   : launch_pair<false, false>(grid2, t.stream, ma, mbh, M, K, nb, bn, per, p,
                                               (size_t)B * M, FusedOut{});
      }
      continue;
    }
    const dim3 grid((M + TC_BM * nsub - 1) / (TC_BM * nsub), used);
    if (fo) {
      FusedOut f = *fo;
      f.n0 = n0;
      launch_variant<true>(transposed, x3, nsub, grid, t.stream, ma, mb, M, K, nb, bn, per,
                           nullptr, 0, f);
    } else {
      // partial sums of this N slab land at part + n0 rows, split stride B x M
      launch_variant<false>(transposed, x3, nsub, grid, t.stream, ma, mb, M, K, nb, bn, per,
                            part + (size_t)n0 * M, (size_t)B * M, FusedOut{});
    }
  }
}

int tc_used_splits(int K, int splits) {
  const int kbs = (K + TC_BK - 1) / TC_BK;
  const int per = (kbs + splits - 1) / splits;
  return (kbs + per - 1) / per;
}

} // namespace xb
