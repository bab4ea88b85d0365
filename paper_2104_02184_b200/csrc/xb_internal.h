// xb_internal.h -- host-side internals shared by the libxbtile translation units.
#pragma once

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/xbtile.h"
#include "xb_common.cuh"

namespace xb {

// error plumbing: every ABI entry catches Err and reports via xb_last_error()
struct Err {
  std::string msg;
};
[[noreturn]] void raise(const std::string &msg);
void set_last_error(const std::string &msg);
// every ABI entry: run f, map exceptions to a non-zero status + xb_last_error()
template <class F> inline int xb_guard(F &&f) {
  try {
    f();
    return 0;
  } catch (const Err &e) {
    set_last_error(e.msg);
    return 1;
  } catch (const std::exception &e) {
    set_last_error(e.what());
    return 1;
  }
}
void cuda_check(cudaError_t e, const char *what);
#define XB_CUDA(call) ::xb::cuda_check((call), #call)
void count_launch(int n = 1);

// the reference's named-stream derivation (proj/src/rng.cpp:14-41)
uint64_t fnv1a(const char *s);
uint64_t splitmix(uint64_t z);
inline uint64_t derive_seed(uint64_t base, const char *name) { return splitmix(base ^ fnv1a(name)); }
// proj/src/rng.cpp:39-41: derive(name, index)
inline uint64_t derive_seed_idx(uint64_t base, const char *name, uint64_t idx) {
  return splitmix(splitmix(base ^ fnv1a(name)) + idx);
}
inline Key key_of(uint64_t seed) { return Key{(uint32_t)seed, (uint32_t)(seed >> 32)}; }

// One-time per-device setup (cudaFuncSetAttribute is per device context): bit
// d of `mask` records that device d is configured.  Concurrent first calls may
// both run f -- harmless, the attributes are idempotent.
inline int current_device() {
  int d = 0;
  XB_CUDA(cudaGetDevice(&d));
  return d;
}
template <class F> inline void once_per_device(std::atomic<uint64_t> &mask, F &&f) {
  const int d = current_device();
  const uint64_t bit = 1ull << (d & 63);
  if (mask.load(std::memory_order_acquire) & bit) return;
  f();
  mask.fetch_or(bit, std::memory_order_acq_rel);
}

// device scratch that grows on demand
struct Scratch {
  void *p = nullptr;
  size_t bytes = 0;
  void *get(size_t n);
  void release();
};

// per-direction converter constants prepared on the host
struct IoDev {
  Quant dac, adc;
  double sigma_inp, sigma_out, sigma_w;
  int nm_absmax, perfect, bm, bm_max_iter;
  // output stage arithmetic: 1 = fp64 like the reference (exact FP32 mode),
  // 0 = fp32 (tensor-core modes, whose accumulators are fp32/TF32 anyway)
  int exact;
};
IoDev make_io(const xb_io_params &io);

// In-stream collectives of a row-sharded tile (xb_comm, xb_comm.cu): NCCL
// over NVLink between processes, or a loopback group of shard handles in one
// process.  Every call is enqueued on `s` and returns without waiting.
struct Collective {
  virtual ~Collective() = default;
  virtual int size() const = 0;
  virtual int rank() const = 0;
  virtual void allreduce_max_i32(int *buf, size_t n, cudaStream_t s) = 0;
  virtual void allreduce_max_f32(float *buf, size_t n, cudaStream_t s) = 0;
  virtual void allreduce_sum_f32(float *buf, size_t n, cudaStream_t s) = 0;
  // the device of this rank's tile, told once when the tile attaches (not a
  // collective, so it may raise: every cross-member check happens here)
  virtual void bind(int device) { (void)device; }
};

// makes `dev` current for the scope of one ABI call on a tile (a handle keeps
// the device it was created on; the caller's current device is restored)
struct DevScope {
  int prev = -1;
  explicit DevScope(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) XB_CUDA(cudaSetDevice(dev));
  }
  ~DevScope() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
  DevScope(const DevScope &) = delete;
  DevScope &operator=(const DevScope &) = delete;
};

struct Tile {
  xb_tile_config cfg;
  int device = 0;            // CUDA device ordinal of every buffer and the stream
  Collective *comm = nullptr; // row shards: the group of the other shards (borrowed)
  cudaStream_t side = nullptr; // backward reductions overlap the next chunk here (lazy)
  std::vector<cudaEvent_t> side_ev; // [2 per backward chunk]
  int R = 0, C = 0;          // local rows, columns
  int row0 = 0, R_total = 0; // first global row, global rows
  int ld = 0;                // leading dimension of W / params (floats)
  uint64_t seed = 0;
  double learning_rate = 0.01;
  Key k_fwd{}, k_bwd{}, k_upd{}, k_c2c{}, k_realize{}, k_temporal{}, k_tinit{};
  uint64_t seq_fwd = 0, seq_bwd = 0, seq_upd = 0; // samples drawn so far per stream
  uint64_t bwd_pending = 0; // samples of backward partials not finished yet (FIFO)
  // device int the pulse kernels read first: nonzero = skip (the host update
  // path points it at the finiteness flag so the weights stay untouched
  // without a host round trip before the launch); nullptr = always run
  const int *abort_flag = nullptr;
  uint32_t upd_calls = 0, temporal_calls = 0;

  float *W = nullptr;      // [R][ld] fp32 weights
  float *Wlo = nullptr;    // [R][ld] compensation terms (comp mode: weight = W + Wlo)
  bool comp = false;       // compensated weights (xb_tile_config.weight_precision)
  // per-cell realization, two planes of [R][ld] float2 in one allocation:
  // steps {dw_up, dw_down} (the pulse kernels), then bounds {w_max, w_min}
  // (every pass that clips: set_weights, temporal, program, drift read 8
  // bytes per cell, not 16)
  float4 *P = nullptr;
  float2 *steps() const { return reinterpret_cast<float2 *>(P); }
  float2 *bounds() const { return reinterpret_cast<float2 *>(P) + (size_t)R * ld; }
  float *xi = nullptr;     // [3][R][ld] temporal d2d draws (lazy)
  float *w0 = nullptr;     // programmed state (lazy)
  float *nu = nullptr;
  double prog_t0 = 0.0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int *bm_count = nullptr; // pinned host word for the bound-management loop
  unsigned *pulse_ctr = nullptr; // pulse kernel's tail work queue {next ticket, warps done}; zero between launches
  int *chk_dev = nullptr;  // input-check flag word (device) and its pinned host copy
  int *chk_host = nullptr;
  float *io_pin = nullptr;  // pinned staging of small host-buffer calls (inputs, then outputs)
  size_t io_pin_n = 0;      // floats
  double *lr_pin = nullptr; // pinned staging of per-sample learning rates
  size_t lr_pin_n = 0;
  cudaEvent_t lr_ev = nullptr; // last lr copy out of lr_pin

  Scratch s_words, s_params, s_io, s_y, s_lr;

  // phase timing (xb_tile_set_timing): pairs of recorded events per phase
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[XB_TIMER_COUNT];
};

// records an event pair around a phase when timing is on
struct PhaseTimer {
  Tile &t;
  int phase;
  cudaEvent_t a = nullptr, b = nullptr;
  PhaseTimer(Tile &t_, int ph);
  ~PhaseTimer();
};

// ---- communicators (xb_comm.cu) ----
struct Collective;
Collective *comm_of(xb_comm *c);

// ---- kernel launchers (xb_update.cu) ----
void launch_rows_amax(const float *V, int B, int n, int ld, float *out, cudaStream_t s);
// one empty kernel (xb_launch_floor_us; not counted as a library launch)
void launch_empty(cudaStream_t s);
// the x and d maxima of an update (rows of length nx and nd) in one launch;
// flag != null: also check_input's finiteness test (bits 1 = x, 2 = d)
void launch_rows_amax2(const float *X, int nx, float *xm, const float *D, int nd, float *dm, int B,
                       cudaStream_t s, int *flag = nullptr);
// per-sample translate + Bernoulli trains; writes packed words and bl[B]
void launch_trains(const Tile &t, const float *X, const float *D, int B, const double *lr_dev,
                   double lr_scalar, const float *xm, const float *dm, uint64_t seq0,
                   uint32_t *xw, uint32_t *dw, int ldb, int32_t *bl, double *px, double *pd,
                   bool deterministic, const double *dwmin_b = nullptr);
// d trains are LINE-major: dw[i][b], row stride ldb (multiple of 8).  x trains
// are QUAD-interleaved: the words of samples 4q..4q+3 of column j form one
// uint4 at quad index q * C + j (xq_index), ldb * C words in all.  A warp of the
// pulse kernel (32 consecutive columns) then reads 4 samples as one coalesced
// 512-byte request instead of 32 separate lines (the L1 data pipe was the
// binding unit with line-major x words).
inline int train_ld(int B) { return (B + 7) / 8 * 8; }
__host__ __device__ inline size_t xq_index(int j, int b, int C) {
  return (((size_t)(b >> 2) * (size_t)C + (size_t)j) << 2) | (size_t)(b & 3);
}
// weight-stationary coincidence/pulse kernel over packed words
// flip inverts every pulse (negative unit-cell gain, tile.cpp:164-167)
// col >= 0: only the 32-column block holding column `col` (x trains zero elsewhere)
void launch_pulse(Tile &t, const uint32_t *xw, const uint32_t *dw, int ldb, int B,
                  uint32_t call_id, bool flip = false, int col = -1);
// Tiki-Taka transfer read (compound.cpp:257-267): out = the forward of the
// one-hot e_col through the output stage of `io` (B = 1, exact fp32 path),
// without a contraction: acc_i = W[i][col] Q_dac(1); also writes e_col [C]
// to onehot.  Only for io without input noise or bound management.
void launch_column_read(Tile &t, int col, const IoDev &io, Key key, uint64_t seq, float *out,
                        float *onehot);
// out[line][k] = in[line][idx[k]] (k < n), zero-padded to ldb_out; quad != 0:
// both sides in the x quad layout (xq_index with C = lines)
void launch_gather_samples(const uint32_t *in, int ldb_in, int lines, const int *idx, int n,
                           uint32_t *out, int ldb_out, cudaStream_t s, bool quad = false);
// W_eff = sum_k g_k W_k over [R][ld] (fp64 sum, fp32 store); K <= XB_MAX_CELL_DEVICES
void launch_effective(float *weff, const float *const *w, const double *g, int K, int R, int C,
                      int ld, cudaStream_t s);
// deterministic_implicit: lround(bl*pd*px) pulses per cell per sample
void launch_pulse_det(Tile &t, const double *px, const double *pd, const int32_t *bl, int B,
                      uint32_t call_id);

// ---- elementwise (xb_elem.cu) ----
void launch_realize(Tile &t);
void launch_clip(Tile &t);
void launch_temporal(Tile &t, const xb_temporal_params &tp, uint32_t call);
void launch_temporal_xi(Tile &t);
void launch_program(Tile &t, const float *target_dev, const xb_inference_model &m, Key key);
void launch_drift(Tile &t, double ratio);
// ORs `bit` into the device word *flag if v[0..n) holds an Inf or NaN
void launch_nonfinite(const float *v, size_t n, int bit, int *flag, cudaStream_t s);

// ---- tcgen05 contraction (xb_mvm_tc.cu) ----
int tc_splits(int M, int K, bool x3);
int tc_used_splits(int K, int splits);
// tc_gemm: declared in xb_mvm_common.cuh (takes the fused output-stage arguments)

// ---- noisy MVM (xb_mvm.cu) ----
// forward: Y[b][i] = alpha_b * ADC(sum_j W[i][j] x~[b][j] + noise), i local rows
void mvm_forward(Tile &t, const float *dX, int B, float *dY, const IoDev &io, Key key,
                 uint64_t seq0);
// backward, unsharded: G[b][j] over all rows
void mvm_backward(Tile &t, const float *dD, int B, float *dG, const IoDev &io, Key key,
                  uint64_t seq0, const float *amax_global, bool partial_only, float *dP);
void mvm_backward_finish(Tile &t, const float *dPsum, int B, const float *amax_global,
                         float *dG, const IoDev &io, Key key, uint64_t seq0);

} // namespace xb
