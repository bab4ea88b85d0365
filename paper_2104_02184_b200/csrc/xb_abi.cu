// xb_abi.cu -- the extern "C" boundary (include/xbtile.h) and the tile handle.
//
// Host-side validation mirrors the reference's error behaviour (messages name
// the field: proj/src/io.cpp:14-30, proj/src/device.cpp:13-24,
// proj/src/pulsed.cpp:13-32, proj/src/tile.cpp:13-23,65-75,103-111); the
// compute runs in the kernels of xb_update.cu / xb_mvm.cu / xb_elem.cu.
#include <atomic>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <initializer_list>

#include "xb_internal.h"

namespace xb {

static thread_local std::string g_err;
static std::atomic<uint64_t> g_launches{0};

void raise(const std::string &msg) { throw Err{msg}; }

void cuda_check(cudaError_t e, const char *what) {
  if (e != cudaSuccess) raise(std::string("CUDA error: ") + cudaGetErrorString(e) + " (" + what + ")");
}

void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

uint64_t fnv1a(const char *s) { // proj/src/rng.cpp:14-21
  uint64_t h = 0xcbf29ce484222325ull;
  for (; *s; ++s) {
    h ^= (unsigned char)*s;
    h *= 0x100000001b3ull;
  }
  return h;
}

uint64_t splitmix(uint64_t z) { // proj/src/rng.cpp:24-29
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

PhaseTimer::PhaseTimer(Tile &t_, int ph) : t(t_), phase(ph) {
  if (!t.timing) return;
  XB_CUDA(cudaEventCreate(&a));
  XB_CUDA(cudaEventCreate(&b));
  XB_CUDA(cudaEventRecord(a, t.stream));
}

PhaseTimer::~PhaseTimer() {
  if (!a) return;
  cudaEventRecord(b, t.stream);
  t.ev[phase].emplace_back(a, b);
}

static void clear_timing(Tile &t) {
  for (auto &v : t.ev) {
    for (auto &p : v) {
      cudaEventDestroy(p.first);
      cudaEventDestroy(p.second);
    }
    v.clear();
  }
}

void *Scratch::get(size_t n) {
  if (n > bytes) {
    if (p) XB_CUDA(cudaFree(p));
    p = nullptr;
    bytes = 0;
    XB_CUDA(cudaMalloc(&p, n));
    bytes = n;
  }
  return p;
}

void Scratch::release() {
  if (p) cudaFree(p);
  p = nullptr;
  bytes = 0;
}

void set_last_error(const std::string &msg) { g_err = msg; }

template <class F> static int guard(F &&f) { return xb_guard(static_cast<F &&>(f)); }

// ------------------------------------------------------------------ validation
static void io_validate(const xb_io_params &io, const char *ctx) { // io.cpp:14-30
  const std::string c(ctx);
  if (io.dac_bits < 0) raise(c + ".dac_bits: must be >= 0");
  if (io.adc_bits < 0) raise(c + ".adc_bits: must be >= 0");
  if (!(io.input_bound > 0.0)) raise(c + ".input_bound: must be > 0");
  if (!(io.output_bound > 0.0)) raise(c + ".output_bound: must be > 0");
  if (io.sigma_inp < 0.0 || io.sigma_out < 0.0 || io.sigma_w < 0.0)
    raise(c + ": noise sigmas must be >= 0");
  if (io.bound_management != XB_BM_NONE && io.bound_management != XB_BM_ITERATIVE)
    raise(c + ".bound_management: unknown mode");
  if (io.bound_management == XB_BM_ITERATIVE && (io.bm_max_iter < 0 || io.bm_max_iter > 30))
    raise(c + ".bm_max_iter: must be in [0, 30]");
}

static void device_validate(const xb_device_params &p, const char *ctx) { // device.cpp:13-24
  const std::string c(ctx);
  if (!(p.dw_min > 0.0)) raise(c + ".dw_min: must be > 0");
  if (!(p.w_min < 0.0 && 0.0 < p.w_max)) raise(c + ": requires w_min < 0 < w_max");
  if (p.dw_min_dtod < 0.0 || p.dw_min_std < 0.0 || p.up_down_dtod < 0.0 || p.w_max_dtod < 0.0 ||
      p.w_min_dtod < 0.0)
    raise(c + ": dtod/std spreads must be >= 0");
  if (p.kind < XB_CONSTANT_STEP || p.kind > XB_EXP_STEP) raise(c + ".kind: unknown device model");
}

static void update_validate(const xb_update_params &u) { // pulsed.cpp:13-17
  if (u.bl < 1) raise("update.bl: must be >= 1");
  if (u.bl > 31) raise("update.bl: must be <= 31 (pulse trains are packed one uint32 per line)");
  if (u.pulse_type != XB_PULSE_STOCHASTIC && u.pulse_type != XB_PULSE_DETERMINISTIC)
    raise("update.pulse_type: unknown");
}

static void temporal_validate(const xb_temporal_params &tp) { // tile.cpp:13-23
  if (tp.decay_rate < 0.0 || tp.diffusion_sigma < 0.0)
    raise("temporal: decay_rate and diffusion_sigma must be >= 0");
  if (tp.reset_prob < 0.0 || tp.reset_prob > 1.0) raise("temporal.reset_prob: must be in [0, 1]");
  if (tp.decay_dtod < 0.0 || tp.diffusion_dtod < 0.0 || tp.reset_dtod < 0.0)
    raise("temporal: dtod spreads must be >= 0");
}

static bool temporal_any(const xb_temporal_params &tp) {
  return tp.decay_rate > 0.0 || tp.diffusion_sigma > 0.0 || tp.reset_prob > 0.0;
}


static void ensure_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    raise("no CUDA device available: the B200 tile has no CPU fallback");
  int dev = 0;
  XB_CUDA(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  XB_CUDA(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10)
    raise(std::string("device ") + prop.name + " is not sm_100 (libxbtile is built for sm_100a only)");
}

static size_t ld_of(int C) { return (size_t)((C + 31) / 32 * 32); }

} // namespace xb

using namespace xb;

struct xb_tile {
  Tile t;
};

struct xb_unitcell {
  xb_unitcell_config cfg;
  xb_tile *eff = nullptr;         // weights-only handle: W_eff and the compound's streams
  std::vector<xb_tile *> members; // all on eff's CUDA stream
  bool dirty = true;              // W_eff stale (compound.cpp:66-80)
  int next_member = 0;            // round-robin cursor, persists across mini-batches
};

struct xb_transfer {
  xb_transfer_config cfg;
  xb_tile *fast = nullptr, *slow = nullptr;
  long counter = 0, events = 0;
  int next_column = 0;
  Scratch onehot, readout, tmp;
};

namespace xb {

static void tile_init_keys(Tile &t, uint64_t seed) {
  t.seed = seed;
  t.k_fwd = key_of(derive_seed(seed, "forward")); // tile.cpp:43-46
  t.k_bwd = key_of(derive_seed(seed, "backward"));
  const uint64_t upd = derive_seed(seed, "update");
  t.k_upd = key_of(upd);
  t.k_c2c = key_of(derive_seed(upd, "c2c"));
  t.k_temporal = key_of(derive_seed(seed, "temporal"));
  t.k_realize = key_of(derive_seed(seed, "realize"));      // tile.cpp:27
  t.k_tinit = key_of(derive_seed(seed, "temporal_init"));  // tile.cpp:59
}

static void tile_alloc(Tile &t) {
  const size_t n = (size_t)t.R * t.ld;
  XB_CUDA(cudaMalloc(&t.W, std::max<size_t>(n, 1) * sizeof(float)));
  XB_CUDA(cudaMalloc(&t.P, std::max<size_t>(n, 1) * sizeof(float4)));
  XB_CUDA(cudaMemsetAsync(t.W, 0, n * sizeof(float), t.stream));
  XB_CUDA(cudaMemsetAsync(t.P, 0, n * sizeof(float4), t.stream));
  if (t.comp) {
    XB_CUDA(cudaMalloc(&t.Wlo, std::max<size_t>(n, 1) * sizeof(float)));
    XB_CUDA(cudaMemsetAsync(t.Wlo, 0, n * sizeof(float), t.stream));
  }
}

// weight writers other than the pulse kernels (set_weights/clip, temporal
// steps, program, drift) act on the fp32 weight and drop the compensation
static void wlo_reset(Tile &t) {
  if (t.comp && t.Wlo)
    XB_CUDA(cudaMemsetAsync(t.Wlo, 0, (size_t)t.R * t.ld * sizeof(float), t.stream));
}

// comp mode: explicit FP32X2, or AUTO when a pulse is under ~2048 fp32 ulps
// of the largest weight the device can hold
static bool want_comp(const xb_tile_config &c) {
  if (c.weight_precision == XB_W_FP32X2) return true;
  if (c.weight_precision == XB_W_FP32) return false;
  const double wb = std::max(std::fabs(c.device.w_max), std::fabs(c.device.w_min)) *
                    (1.0 + 3.0 * std::max(c.device.w_max_dtod, c.device.w_min_dtod));
  return c.device.dw_min < std::ldexp(wb, -12);
}

static void tile_free(Tile &t) {
  clear_timing(t);
  cudaFree(t.W);
  cudaFree(t.Wlo);
  cudaFree(t.P);
  cudaFree(t.xi);
  cudaFree(t.w0);
  cudaFree(t.nu);
  t.s_words.release();
  t.s_params.release();
  t.s_io.release();
  t.s_y.release();
  t.s_lr.release();
  if (t.own_stream && t.stream) cudaStreamDestroy(t.stream);
  if (t.bm_count) cudaFreeHost(t.bm_count);
  if (t.chk_host) cudaFreeHost(t.chk_host);
  if (t.lr_pin) cudaFreeHost(t.lr_pin);
  if (t.io_pin) cudaFreeHost(t.io_pin);
  if (t.lr_ev) cudaEventDestroy(t.lr_ev);
  for (cudaEvent_t e : t.side_ev) cudaEventDestroy(e);
  if (t.side) cudaStreamDestroy(t.side);
  cudaFree(t.chk_dev);
  cudaFree(t.pulse_ctr);
}

static void sync(Tile &t) { XB_CUDA(cudaStreamSynchronize(t.stream)); }

// Small host-buffer calls -- the per-sample reference API -- stage their
// inputs and outputs through one pinned buffer per tile: a pageable copy
// costs the driver a staging pass and several microseconds more latency each
// way, a pinned one is a plain DMA.  Every host-buffer entry synchronises
// the tile's stream before it returns, so the buffer is free at the next call.
constexpr size_t kPinStageMax = size_t(1) << 18; // floats per call (1 MB)

static float *io_stage(Tile &t, size_t n) {
  if (n == 0 || n > kPinStageMax) return nullptr;
  if (t.io_pin_n < n) {
    if (t.io_pin) XB_CUDA(cudaFreeHost(t.io_pin));
    t.io_pin = nullptr;
    t.io_pin_n = 0;
    const size_t want = std::max<size_t>(n, 8192);
    XB_CUDA(cudaMallocHost(&t.io_pin, want * sizeof(float)));
    t.io_pin_n = want;
  }
  return t.io_pin;
}

// host -> device of n floats, through `pin` (a slot of io_stage) when given
static void h2d(Tile &t, float *dst, const float *src, size_t n, float *pin) {
  if (pin) {
    std::memcpy(pin, src, n * sizeof(float));
    src = pin;
  }
  XB_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(float), cudaMemcpyHostToDevice, t.stream));
}

// device -> host of n floats and the stream sync that ends a host-buffer call
static void d2h_sync(Tile &t, float *dst, const float *src, size_t n, float *pin) {
  XB_CUDA(cudaMemcpyAsync(pin ? pin : dst, src, n * sizeof(float), cudaMemcpyDeviceToHost,
                          t.stream));
  sync(t);
  if (pin) std::memcpy(dst, pin, n * sizeof(float));
}

// check_input's finiteness test (tile.cpp:65-75) on the inputs after their
// H2D copy: one streaming kernel per array on the tile's stream, then one
// 4-byte read.  Raises with the reference's message, naming the first bad
// array in argument order, before any state of the tile changes.
struct Finite {
  const float *v;
  size_t n;
  const char *what;
};
// the input-check flag word, cleared in stream order
static void clear_chk(Tile &t) {
  if (!t.chk_dev) {
    XB_CUDA(cudaMalloc(&t.chk_dev, sizeof(int)));
    XB_CUDA(cudaMallocHost(&t.chk_host, sizeof(int)));
  }
  XB_CUDA(cudaMemsetAsync(t.chk_dev, 0, sizeof(int), t.stream));
}

// launch half: the flag bits land in t.chk_dev (stream order), nothing waits
static void launch_finite_dev(Tile &t, std::initializer_list<Finite> arrays) {
  clear_chk(t);
  int bit = 1;
  for (const Finite &a : arrays) {
    launch_nonfinite(a.v, a.n, bit, t.chk_dev, t.stream);
    bit <<= 1;
  }
}

// read half: one 4-byte read and a stream sync; raises for the first bad array
static void raise_if_nonfinite(Tile &t, std::initializer_list<Finite> arrays) {
  XB_CUDA(cudaMemcpyAsync(t.chk_host, t.chk_dev, sizeof(int), cudaMemcpyDeviceToHost, t.stream));
  sync(t);
  int bit = 1;
  for (const Finite &a : arrays) {
    if (*t.chk_host & bit) raise(std::string(a.what) + ": non-finite entry");
    bit <<= 1;
  }
}

static void check_finite_dev(Tile &t, std::initializer_list<Finite> arrays) {
  launch_finite_dev(t, arrays);
  raise_if_nonfinite(t, arrays);
}

// Small host inputs (cfg1/cfg2-sized calls) are scanned on the host before
// the copy: cheaper than a kernel, a 4-byte read and a stream sync.  Same
// test (exponent all ones = Inf/NaN), same order, same messages.
constexpr size_t kHostCheckMax = size_t(1) << 16; // floats over all arrays of a call

static bool host_check_small(std::initializer_list<Finite> host_arrays) {
  size_t n = 0;
  for (const Finite &a : host_arrays) n += a.n;
  if (n > kHostCheckMax) return false;
  for (const Finite &a : host_arrays) {
    const uint32_t *u = reinterpret_cast<const uint32_t *>(a.v);
    uint32_t bad = 0;
    for (size_t i = 0; i < a.n; ++i) bad |= ((u[i] & 0x7f800000u) == 0x7f800000u);
    if (bad) raise(std::string(a.what) + ": non-finite entry");
  }
  return true;
}

static void ensure_xi(Tile &t) {
  if (t.xi) return;
  XB_CUDA(cudaMalloc(&t.xi, std::max<size_t>(3 * (size_t)t.R * t.ld, 1) * sizeof(float)));
  launch_temporal_xi(t);
}

// ---- host-buffer staging ----
struct Staged {
  float *a = nullptr, *b = nullptr;
};

template <class T> static T *scratch_as(Scratch &s, size_t count) {
  return (T *)s.get(std::max<size_t>(count, 1) * sizeof(T));
}

// validate a host lr array the way the reference does per sample: lr == 0 or
// a zero vector is a no-op; otherwise lr must be > 0 (pulsed.cpp:27-29,122-124)
static void check_lr_host(const float *X, const float *D, int B, int C, int R, const double *lr,
                          double def_lr) {
  for (int b = 0; b < B; ++b) {
    const double l = lr ? lr[b] : def_lr;
    if (l == 0.0) continue;
    bool xz = true, dz = true;
    for (int j = 0; j < C && xz; ++j) xz = X[(size_t)b * C + j] == 0.f;
    for (int i = 0; i < R && dz; ++i) dz = D[(size_t)b * R + i] == 0.f;
    if (xz || dz) continue;
    if (!(l > 0.0)) raise("translate: learning rate must be > 0");
  }
}

static void check_lr_dev(const double *lr, int B, double def_lr) {
  for (int b = 0; b < B; ++b) {
    const double l = lr ? lr[b] : def_lr;
    if (!(l >= 0.0)) raise("translate: learning rate must be > 0");
  }
}

// update scratch layout
struct UpdBufs {
  double *lr;
  float *xm, *dm;
  int32_t *bl;
  uint32_t *xw, *dw;
  double *px, *pd;
};

static UpdBufs upd_bufs(Tile &t, int B, bool det) {
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t s_lr = al(B * sizeof(double)), s_bl = al(B * sizeof(int32_t));
  const size_t nb = det ? (size_t)B : (size_t)train_ld(B); // ldb words per line (x quads, d lines)
  const size_t s_xw = al(nb * t.C * (det ? sizeof(double) : sizeof(uint32_t)));
  const size_t s_dw = al(nb * std::max(t.R, 1) * (det ? sizeof(double) : sizeof(uint32_t)));
  char *p = (char *)t.s_words.get(3 * s_lr + s_bl + s_xw + s_dw);
  UpdBufs u{};
  u.lr = (double *)p;
  u.xm = (float *)(p + s_lr);
  u.dm = (float *)(p + 2 * s_lr);
  u.bl = (int32_t *)(p + 3 * s_lr);
  char *q = p + 3 * s_lr + s_bl;
  if (det) {
    u.px = (double *)q;
    u.pd = (double *)(q + s_xw);
  } else {
    u.xw = (uint32_t *)q;
    u.dw = (uint32_t *)(q + s_xw);
  }
  return u;
}

// a uniform learning rate travels as a kernel argument (no copy, no sync);
// per-sample rates are staged in the tile's pinned buffer (the host array is
// only borrowed for the call) and copied in stream order.  The staging buffer
// is reused only after its previous copy has executed (an event, not a
// stream sync).
static const double *upload_lr(Tile &t, double *dst, const double *lr, int B, double *scalar) {
  *scalar = lr ? lr[0] : t.learning_rate;
  bool uniform = true;
  for (int b = 1; lr && b < B && uniform; ++b) uniform = lr[b] == lr[0];
  if (uniform) return nullptr;
  if (t.lr_ev) XB_CUDA(cudaEventSynchronize(t.lr_ev));
  if (t.lr_pin_n < (size_t)B) {
    if (t.lr_pin) XB_CUDA(cudaFreeHost(t.lr_pin));
    t.lr_pin = nullptr;
    t.lr_pin_n = 0;
    XB_CUDA(cudaMallocHost(&t.lr_pin, (size_t)B * sizeof(double)));
    t.lr_pin_n = (size_t)B;
  }
  if (!t.lr_ev) XB_CUDA(cudaEventCreateWithFlags(&t.lr_ev, cudaEventDisableTiming));
  std::memcpy(t.lr_pin, lr, (size_t)B * sizeof(double));
  XB_CUDA(cudaMemcpyAsync(dst, t.lr_pin, B * sizeof(double), cudaMemcpyHostToDevice, t.stream));
  XB_CUDA(cudaEventRecord(t.lr_ev, t.stream));
  return dst;
}

// the whole pulsed update of B samples from device inputs
static void update_device(Tile &t, const float *dX, const float *dD, int B, const double *lr,
                          const float *dAmaxD, bool peek, uint32_t *xw_out, uint32_t *dw_out,
                          int32_t *bl_out, int col = -1) {
  const bool det = t.cfg.update.pulse_type == XB_PULSE_DETERMINISTIC && !peek;
  UpdBufs u = upd_bufs(t, B, det);
  double lr_s = 0.0;
  const double *lr_d = upload_lr(t, u.lr, lr, B, &lr_s);
  {
    PhaseTimer pt(t, XB_TIMER_TRAINS);
    const float *dm = dAmaxD;
    if (!dm) {
      // (abort_flag set: the host-buffer update's finiteness test rides along)
      launch_rows_amax2(dX, t.C, u.xm, dD, t.R, u.dm, B, t.stream,
                        t.abort_flag ? t.chk_dev : nullptr);
      // row shard: translate needs max|d| over the whole tile (pulsed.cpp:34-51)
      if (t.comm) t.comm->allreduce_max_f32(u.dm, (size_t)B, t.stream);
      dm = u.dm;
    } else {
      launch_rows_amax(dX, B, t.C, t.C, u.xm, t.stream);
    }
    launch_trains(t, dX, dD, B, lr_d, lr_s, u.xm, dm, t.seq_upd, u.xw, u.dw, train_ld(B), u.bl,
                  u.px, u.pd, det);
  }
  if (peek) { // back to the reference-facing sample-major layout
    const int ldb = train_ld(B);
    std::vector<uint32_t> hx((size_t)ldb * t.C), hd((size_t)ldb * t.R);
    XB_CUDA(cudaMemcpyAsync(hx.data(), u.xw, sizeof(uint32_t) * hx.size(),
                            cudaMemcpyDeviceToHost, t.stream));
    XB_CUDA(cudaMemcpyAsync(hd.data(), u.dw, sizeof(uint32_t) * hd.size(),
                            cudaMemcpyDeviceToHost, t.stream));
    XB_CUDA(cudaMemcpyAsync(bl_out, u.bl, sizeof(int32_t) * B, cudaMemcpyDeviceToHost, t.stream));
    sync(t);
    for (int b = 0; b < B; ++b) {
      for (int j = 0; j < t.C; ++j) xw_out[(size_t)b * t.C + j] = hx[xq_index(j, b, t.C)];
      for (int i = 0; i < t.R; ++i) dw_out[(size_t)b * t.R + i] = hd[(size_t)i * ldb + b];
    }
    return;
  }
  {
    PhaseTimer pt(t, XB_TIMER_PULSE);
    if (det)
      launch_pulse_det(t, u.px, u.pd, u.bl, B, t.upd_calls);
    else
      launch_pulse(t, u.xw, u.dw, train_ld(B), B, t.upd_calls, false, col);
  }
  t.upd_calls += 1;
  t.seq_upd += (uint64_t)B;
}

static void forward_device(Tile &t, const float *dX, int B, float *dY, const xb_io_params &io) {
  io_validate(io, "forward_io");
  PhaseTimer pt(t, XB_TIMER_FORWARD);
  mvm_forward(t, dX, B, dY, make_io(io), t.k_fwd, t.seq_fwd);
  t.seq_fwd += (uint64_t)B;
}

static xb_io_params noisy_io(const xb_io_params &io, double extra) { // io.cpp:74-91
  xb_io_params out = io;
  if (extra <= 0.0) return out;
  if (out.is_perfect) {
    xb_default_io(&out);
    out.dac_bits = 0;
    out.adc_bits = 0;
    out.input_bound = INFINITY;
    out.output_bound = INFINITY;
    out.sigma_out = 0.0;
    out.noise_management = XB_NM_NONE;
  }
  out.is_perfect = 0;
  out.sigma_w = std::hypot(out.sigma_w, extra);
  return out;
}

} // namespace xb

extern "C" {

int xb_abi_version(void) { return XB_ABI_VERSION; }
const char *xb_last_error(void) { return g_err.c_str(); }
uint64_t xb_launch_count(void) { return g_launches.load(); }

int xb_launch_floor_us(int n, int reps, double *us_per_launch) {
  return guard([&] {
    if (n < 1 || reps < 1) raise("launch_floor: need n >= 1 and reps >= 1");
    ensure_device();
    cudaStream_t s;
    cudaEvent_t e0, e1;
    XB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    XB_CUDA(cudaEventCreate(&e0));
    XB_CUDA(cudaEventCreate(&e1));
    float best = 0.f;
    for (int r = 0; r <= reps; ++r) { // round 0 warms up
      XB_CUDA(cudaEventRecord(e0, s));
      for (int k = 0; k < n; ++k) launch_empty(s);
      XB_CUDA(cudaEventRecord(e1, s));
      XB_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      XB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      if (r > 0 && (r == 1 || ms < best)) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s);
    *us_per_launch = 1e3 * (double)best / n;
  });
}

int xb_device_check(void) {
  return guard([] { ensure_device(); });
}

void xb_default_device(xb_device_params *p) { // device.hpp:24-39
  std::memset(p, 0, sizeof *p);
  p->kind = XB_CONSTANT_STEP;
  p->dw_min = 0.001;
  p->w_max = 1.0;
  p->w_min = -1.0;
  p->slope = 1.0;
  p->gamma = 2.0;
}

void xb_default_io(xb_io_params *p) { // io.hpp:21-33
  std::memset(p, 0, sizeof *p);
  p->dac_bits = 7;
  p->adc_bits = 9;
  p->input_bound = 1.0;
  p->output_bound = 12.0;
  p->sigma_out = 0.06;
  p->noise_management = XB_NM_ABS_MAX;
  p->bound_management = XB_BM_NONE;
  p->bm_max_iter = 10;
}

void xb_perfect_io(xb_io_params *p) { // io.cpp:32-40
  xb_default_io(p);
  p->is_perfect = 1;
  p->dac_bits = 0;
  p->adc_bits = 0;
  p->sigma_out = 0.0;
  p->noise_management = XB_NM_NONE;
}

void xb_default_config(xb_tile_config *c) {
  std::memset(c, 0, sizeof *c);
  xb_default_device(&c->device);
  xb_default_io(&c->forward_io);
  xb_default_io(&c->backward_io);
  c->update.bl = 31;
  c->update.bl_management = 0;
  c->update.pulse_type = XB_PULSE_STOCHASTIC;
  c->mvm_precision = XB_MVM_TF32X3;
}

void xb_default_transfer_config(xb_transfer_config *c) { // compound.hpp:76-91
  std::memset(c, 0, sizeof *c);
  xb_default_device(&c->fast_device);
  xb_default_device(&c->slow_device);
  xb_default_io(&c->forward_io);
  xb_default_io(&c->backward_io);
  c->update.bl = 31;
  c->mvm_precision = XB_MVM_TF32X3;
  c->transfer_every = 1;
  c->units_in_mbatch = 0;
  c->transfer_lr = 0.1;
  c->columns_per_event = 1;
  c->gamma = 0.0;
  c->has_transfer_io = 0;
  xb_default_io(&c->transfer_io);
}

void xb_default_inference_model(xb_inference_model *m) { // inference.hpp:21-36
  std::memset(m, 0, sizeof *m);
  m->prog_noise_scale = 1.0;
  m->prog_c0 = 0.26;
  m->prog_c1 = 1.66;
  m->prog_c2 = 0.33;
  m->nu_mean = 0.06;
  m->nu_std = 0.03;
  m->t0 = 20.0;
  m->nu_min = 0.0;
  m->nu_max = 1.0;
  m->compensation_probes = 10;
}

int xb_device_preset(const char *name, xb_device_params *p) { // device.cpp:100-132
  return guard([&] {
    xb_default_device(p);
    const std::string n(name ? name : "");
    if (n == "ideal") {
      p->kind = XB_CONSTANT_STEP;
      p->dw_min = 1e-6;
      return;
    }
    if (n == "reram_sb") {
      p->kind = XB_SOFT_BOUNDS;
      p->dw_min = 0.002;
      p->dw_min_dtod = 0.3;
      p->dw_min_std = 0.3;
      p->w_max = 0.6;
      p->w_min = -0.6;
      p->up_down_dtod = 0.01;
      return;
    }
    if (n == "reram_es") {
      p->kind = XB_EXP_STEP;
      p->dw_min = 0.001;
      p->dw_min_dtod = 0.3;
      p->dw_min_std = 0.3;
      p->w_max = 0.6;
      p->w_min = -0.6;
      p->up_down = 0.1;
      p->up_down_dtod = 0.01;
      p->gamma = 2.0;
      return;
    }
    raise("device preset: unknown name '" + n + "'");
  });
}

int xb_tile_create(const xb_tile_config *cfg, int d_out, int d_in, uint64_t seed,
                   const xb_shard *shard, xb_tile **out) {
  return guard([&] {
    *out = nullptr;
    if (d_out < 1 || d_in < 1) raise("tile: dimensions must be >= 1"); // tile.cpp:47-49
    io_validate(cfg->forward_io, "forward_io");
    io_validate(cfg->backward_io, "backward_io");
    update_validate(cfg->update);
    temporal_validate(cfg->temporal);
    device_validate(cfg->device, "device");
    if (cfg->mvm_precision != XB_MVM_FP32 && cfg->mvm_precision != XB_MVM_TF32 &&
        cfg->mvm_precision != XB_MVM_TF32X3)
      raise("mvm_precision: unknown mode");
    if (cfg->weight_precision < XB_W_AUTO || cfg->weight_precision > XB_W_FP32X2)
      raise("weight_precision: unknown mode");
    int r0 = 0, r1 = d_out;
    if (shard) {
      if (shard->d_out_total != d_out) raise("shard.d_out_total: must equal d_out");
      r0 = shard->row_begin;
      r1 = shard->row_end;
      if (r0 < 0 || r1 > d_out || r0 >= r1) raise("shard: need 0 <= row_begin < row_end <= d_out");
    }
    ensure_device();
    auto h = std::make_unique<xb_tile>();
    Tile &t = h->t;
    DevScope ds_(t.device);
    t.cfg = *cfg;
    t.R = r1 - r0;
    t.C = d_in;
    t.row0 = r0;
    t.R_total = d_out;
    t.ld = (int)ld_of(d_in);
    t.comp = want_comp(*cfg);
    t.device = current_device();
    XB_CUDA(cudaStreamCreateWithFlags(&t.stream, cudaStreamNonBlocking));
    t.own_stream = true;
    tile_init_keys(t, seed);
    try {
      tile_alloc(t);
      launch_realize(t); // device.cpp:79-88 (Philox realization; upload for parity)
      if (temporal_any(cfg->temporal)) ensure_xi(t);
      sync(t);
    } catch (...) {
      tile_free(t);
      throw;
    }
    *out = h.release();
  });
}

int xb_tile_destroy(xb_tile *t) {
  return guard([&] {
    if (!t) return;
    cudaStreamSynchronize(t->t.stream);
    tile_free(t->t);
    delete t;
  });
}

int xb_tile_clone(const xb_tile *src, xb_tile **out) { // tile.hpp:91 (deep copy)
  return guard([&] {
    *out = nullptr;
    const Tile &s = src->t;
    DevScope ds(s.device);
    XB_CUDA(cudaStreamSynchronize(s.stream));
    auto h = std::make_unique<xb_tile>();
    Tile &t = h->t;
    DevScope ds_(t.device);
    t.cfg = s.cfg;
    t.R = s.R;
    t.C = s.C;
    t.row0 = s.row0;
    t.R_total = s.R_total;
    t.ld = s.ld;
    t.learning_rate = s.learning_rate;
    t.seq_fwd = s.seq_fwd;
    t.seq_bwd = s.seq_bwd;
    t.bwd_pending = s.bwd_pending;
    t.seq_upd = s.seq_upd;
    t.upd_calls = s.upd_calls;
    t.temporal_calls = s.temporal_calls;
    t.prog_t0 = s.prog_t0;
    tile_init_keys(t, s.seed);
    t.comp = s.comp;
    t.device = s.device;
    XB_CUDA(cudaStreamCreateWithFlags(&t.stream, cudaStreamNonBlocking));
    t.own_stream = true;
    try {
      tile_alloc(t);
      const size_t n = (size_t)t.R * t.ld;
      XB_CUDA(cudaMemcpyAsync(t.W, s.W, n * sizeof(float), cudaMemcpyDeviceToDevice, t.stream));
      if (t.comp)
        XB_CUDA(cudaMemcpyAsync(t.Wlo, s.Wlo, n * sizeof(float), cudaMemcpyDeviceToDevice,
                                t.stream));
      XB_CUDA(cudaMemcpyAsync(t.P, s.P, n * sizeof(float4), cudaMemcpyDeviceToDevice, t.stream));
      if (s.xi) {
        XB_CUDA(cudaMalloc(&t.xi, 3 * n * sizeof(float)));
        XB_CUDA(cudaMemcpyAsync(t.xi, s.xi, 3 * n * sizeof(float), cudaMemcpyDeviceToDevice,
                                t.stream));
      }
      if (s.w0) {
        XB_CUDA(cudaMalloc(&t.w0, n * sizeof(float)));
        XB_CUDA(cudaMalloc(&t.nu, n * sizeof(float)));
        XB_CUDA(cudaMemcpyAsync(t.w0, s.w0, n * sizeof(float), cudaMemcpyDeviceToDevice, t.stream));
        XB_CUDA(cudaMemcpyAsync(t.nu, s.nu, n * sizeof(float), cudaMemcpyDeviceToDevice, t.stream));
      }
      sync(t);
    } catch (...) {
      tile_free(t);
      throw;
    }
    *out = h.release();
  });
}

int xb_tile_shape(const xb_tile *t, int *d_out_local, int *d_in, int *row_begin,
                  int *d_out_total) {
  if (d_out_local) *d_out_local = t->t.R;
  if (d_in) *d_in = t->t.C;
  if (row_begin) *row_begin = t->t.row0;
  if (d_out_total) *d_out_total = t->t.R_total;
  return 0;
}

int xb_tile_set_stream(xb_tile *h, void *stream) {
  return guard([&] {
    Tile &t = h->t;
    DevScope ds_(t.device);
    XB_CUDA(cudaStreamSynchronize(t.stream));
    if (t.own_stream) XB_CUDA(cudaStreamDestroy(t.stream));
    if (stream) {
      t.stream = (cudaStream_t)stream;
      t.own_stream = false;
    } else {
      XB_CUDA(cudaStreamCreateWithFlags(&t.stream, cudaStreamNonBlocking));
      t.own_stream = true;
    }
  });
}

void *xb_tile_stream(const xb_tile *t) { return (void *)t->t.stream; }

int xb_tile_synchronize(xb_tile *t) {
  return guard([&] { sync(t->t); });
}

int xb_tile_set_timing(xb_tile *h, int enable) {
  return guard([&] {
    sync(h->t);
    clear_timing(h->t);
    h->t.timing = enable != 0;
  });
}

int xb_tile_read_timing(xb_tile *h, double *ms, int *counts) {
  return guard([&] {
    Tile &t = h->t;
    DevScope ds_(t.device);
    sync(t);
    for (int k = 0; k < XB_TIMER_COUNT; ++k) {
      double tot = 0.0;
      for (auto &p : t.ev[k]) {
        float e = 0.f;
        XB_CUDA(cudaEventElapsedTime(&e, p.first, p.second));
        tot += e;
      }
      if (ms) ms[k] = tot;
      if (counts) counts[k] = (int)t.ev[k].size();
    }
    clear_timing(t);
  });
}

int xb_tile_set_weights(xb_tile *h, const float *w) { // tile.cpp:103-119
  return guard([&] {
    Tile &t = h->t;
    DevScope ds_(t.device);
    XB_CUDA(cudaMemcpy2DAsync(t.W, t.ld * sizeof(float), w, t.C * sizeof(float),
                              t.C * sizeof(float), t.R, cudaMemcpyHostToDevice, t.stream));
    launch_clip(t);
    wlo_reset(t);
    sync(t);
  });
}

int xb_tile_get_weights(const xb_tile *h, float *w) {
  return guard([&] {
    const Tile &t = h->t;
    DevScope ds_(t.device);
    XB_CUDA(cudaMemcpy2DAsync(w, t.C * sizeof(float), t.W, t.ld * sizeof(float),
                              t.C * sizeof(float), t.R, cudaMemcpyDeviceToHost, t.stream));
    XB_CUDA(cudaStreamSynchronize(t.stream));
  });
}

int xb_tile_set_device(xb_tile *h, const float *dw_up, const float *dw_down, const float *w_max,
                       const float *w_min) {
  return guard([&] {
    Tile &t = h->t;
    DevScope ds_(t.device);
    const size_t n = (size_t)t.R * t.ld;
    std::vector<float2> p(2 * n); // planes: steps [n], bounds [n] (Tile::P)
    XB_CUDA(cudaStreamSynchronize(t.stream));
    XB_CUDA(cudaMemcpy(p.data(), t.P, 2 * n * sizeof(float2), cudaMemcpyDeviceToHost));
    for (int i = 0; i < t.R; ++i) {
      for (int j = 0; j < t.C; ++j) {
        const size_t s = (size_t)i * t.C + j, k = (size_t)i * t.ld + j;
        float2 &st = p[k], &bd = p[n + k];
        if (dw_up) st.x = dw_up[s];
        if (dw_down) st.y = dw_down[s];
        if (w_max) bd.x = w_max[s];
        if (w_min) bd.y = w_min[s];
        if (!(bd.y < 0.f && 0.f < bd.x)) raise("set_device: requires w_min < 0 < w_max per cell");
      }
    }
    XB_CUDA(cudaMemcpy(t.P, p.data(), 2 * n * sizeof(float2), cudaMemcpyHostToDevice));
    launch_clip(t);
    wlo_reset(t);
    sync(t);
  });
}

int xb_tile_get_device(const xb_tile *h, float *dw_up, float *dw_down, float *w_max,
                       float *w_min) {
  return guard([&] {
    const Tile &t = h->t;
    DevScope ds_(t.device);
    const size_t n = (size_t)t.R * t.ld;
    std::vector<float2> p(2 * n); // planes: steps [n], bounds [n] (Tile::P)
    XB_CUDA(cudaStreamSynchronize(t.stream));
    XB_CUDA(cudaMemcpy(p.data(), t.P, 2 * n * sizeof(float2), cudaMemcpyDeviceToHost));
    for (int i = 0; i < t.R; ++i) {
      for (int j = 0; j < t.C; ++j) {
        const size_t s = (size_t)i * t.C + j, k = (size_t)i * t.ld + j;
        if (dw_up) dw_up[s] = p[k].x;
        if (dw_down) dw_down[s] = p[k].y;
        if (w_max) w_max[s] = p[n + k].x;
        if (w_min) w_min[s] = p[n + k].y;
      }
    }
  });
}

int xb_tile_forward_dev(xb_tile *h, const float *dX, int B, float *dY, const xb_io_params *io,
                        double extra_sigma) {
  return guard([&] {
    Tile &t = h->t;
    DevScope ds_(t.device);
    if (B < 0) raise("forward: batch must be >= 0");
    const xb_io_params base = io ? *io : t.cfg.forward_io;
    forward_device(t, dX, B, dY, noisy_io(base, extra_sigma));
  });
}

// check = false: callers without check_input (the unit cell, compound.cpp:82-107)
static void forward_host(xb_tile *h, const float *X, int B, float *Y, const xb_io_params &io,
                         bool check = true) {
  Tile &t = h->t;
  DevScope ds_(t.device);
  if (B < 0) raise("forward: batch must be >= 0");
  if (B == 0) return;
  float *dX = scratch_as<float>(t.s_y, (size_t)B * (t.C + t.R));
  float *dY = dX + (size_t)B * t.C;
  const bool checked = !check || host_check_small({{X, (size_t)B * t.C, "forward"}});
  const size_t nx = (size_t)B * t.C, ny = (size_t)B * t.R;
  float *pin = io_stage(t, nx + ny);
  h2d(t, dX, X, nx, pin);
  // large inputs: the finiteness scan is enqueued ahead of the forward and its
  // flag read back with the outputs -- one host round trip per call, not two;
  // a non-finite input rolls the noise counter back and raises (the output
  // buffer is then unspecified, as for every failed call)
  if (!checked) launch_finite_dev(t, {{dX, nx, "forward"}});
  const uint64_t seq = t.seq_fwd;
  forward_device(t, dX, B, dY, io);
  if (!checked)
    XB_CUDA(cudaMemcpyAsync(t.chk_host, t.chk_dev, sizeof(int), cudaMemcpyDeviceToHost, t.stream));
  d2h_sync(t, Y, dY, ny, pin ? pin + nx : nullptr);
  if (!checked && (*t.chk_host & 1)) {
    t.seq_fwd = seq;
    raise("forward: non-finite entry");
  }
}

int xb_tile_forward(xb_tile *h, const float *X, int B, float *Y) {
  return guard([&] { forward_host(h, X, B, Y, h->t.cfg.forward_io); });
}

int xb_tile_forward_io(xb_tile *h, const float *X, int B, float *Y, const xb_io_params *io) {
  return guard([&] { forward_host(h, X, B, Y, *io); });
}

int xb_tile_forward_noisy(xb_tile *h, const float *X, int B, float *Y, double extra_sigma) {
  return guard([&] { forward_host(h, X, B, Y, noisy_io(h->t.cfg.forward_io, extra_sigma)); });
}

// Backward of a row shard with an attached communicator: the global max|d|
// (all-reduce max), then per sample chunk the shard's column sums (partial),
// their all-reduce(sum) on the side stream -- overlapping the next chunk's
// contraction on the tile stream -- and the output stage on the reduced sums
// (finish), in chunk order.  Noise draws are addressed by sample: the result
// does not depend on the chunking.
static void backward_sharded(Tile &t, const float *dD, int B, float *dG) {
  if (B <= 0) return;
  const xb_io_params &io = t.cfg.backward_io;
  if (io.bound_management != XB_BM_NONE)
    raise("backward_io.bound_management: not supported on row shards");
  io_validate(io, "backward_io");
  const int nch = B >= 256 ? 4 : 1;
  const size_t amax_b = ((size_t)B * sizeof(float) + 255) & ~(size_t)255;
  char *p = (char *)t.s_y.get(amax_b + (size_t)B * t.C * sizeof(float) + 256);
  float *amax = (float *)p;
  float *P = (float *)(p + amax_b);
  launch_rows_amax(dD, B, t.R, t.R, amax, t.stream);
  t.comm->allreduce_max_f32(amax, (size_t)B, t.stream);
  if (!t.side) XB_CUDA(cudaStreamCreateWithFlags(&t.side, cudaStreamNonBlocking));
  while ((int)t.side_ev.size() < 2 * nch) {
    cudaEvent_t e;
    XB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    t.side_ev.push_back(e);
  }
  const IoDev d = make_io(io);
  std::vector<int> edge(nch + 1);
  for (int k = 0; k <= nch; ++k) edge[k] = (int)((long)B * k / nch);
  for (int k = 0; k < nch; ++k) {
    const int b0 = edge[k], nb = edge[k + 1] - b0;
    float *Pk = P + (size_t)b0 * t.C;
    mvm_backward(t, dD + (size_t)b0 * t.R, nb, nullptr, d, t.k_bwd, t.seq_bwd + t.bwd_pending,
                 amax + b0, true, Pk);
    t.bwd_pending += (uint64_t)nb;
    XB_CUDA(cudaEventRecord(t.side_ev[2 * k], t.stream));
    XB_CUDA(cudaStreamWaitEvent(t.side, t.side_ev[2 * k], 0));
    t.comm->allreduce_sum_f32(Pk, (size_t)nb * t.C, t.side);
    XB_CUDA(cudaEventRecord(t.side_ev[2 * k + 1], t.side));
  }
  for (int k = 0; k < nch; ++k) {
    const int b0 = edge[k], nb = edge[k + 1] - b0;
    XB_CUDA(cudaStreamWaitEvent(t.stream, t.side_ev[2 * k + 1], 0));
    mvm_backward_finish(t, P + (size_t)b0 * t.C, nb, amax + b0, dG + (size_t)b0 * t.C, d, t.k_bwd,
                        t.seq_bwd);
    t.seq_bwd += (uint64_t)nb;
    t.bwd_pending -= std::min(t.bwd_pending, (uint64_t)nb);
  }
}

int xb_tile_backward_dev(xb_tile *h, const float *dD, int B, float *dG) {
  return guard([&] {
    Tile &t = h->t;
    DevScope ds_(t.device);
    if (t.R != t.R_total && t.comm) return backward_sharded(t, dD, B, dG);
    if (t.R != t.R_total) raise("backward: row-sharded tile; use xb_tile_backward_partial_dev");
    io_validate(t.cfg.backward_io, "backward_io");
    mvm_backward(t, dD, B, dG, make_io(t.cfg.backward_io), t.k_bwd, t.seq_bwd, nullptr, false,
                 nullptr);
    t.seq_bwd += (uint64_t)B;
  });
}

static void backward_host(xb_tile *h, const float *D, int B, float *G, bool check = true) {
  Tile &t = h->t;
  DevScope ds_(t.device);
  if (B < 0) raise("backward: batch must be >= 0");
  if (B == 0) return;
  const bool sharded = t.R != t.R_total;
  if (sharded && !t.comm)
    raise("backward: row-sharded tile; attach a communicator (xb_tile_attach_comm) or use "
          "xb_tile_backward_partial_dev");
  // sharded: D and G live in s_params (backward_sharded uses s_y for its scratch)
  float *dD = sharded ? scratch_as<float>(t.s_params, (size_t)B * (t.C + t.R))
                      : scratch_as<float>(t.s_y, (size_t)B * (t.C + t.R));
  float *dG = dD + (size_t)B * t.R;
  const bool checked = !check || host_check_small({{D, (size_t)B * t.R, "backward"}});
  const size_t nd = (size_t)B * t.R, ng = (size_t)B * t.C;
  float *pin = io_stage(t, nd + ng);
  h2d(t, dD, D, nd, pin);
  if (!checked) check_finite_dev(t, {{dD, nd, "backward"}});
  if (sharded) {
    backward_sharded(t, dD, B, dG);
    d2h_sync(t, G, dG, ng, pin ? pin + nd : nullptr);
    return;
  }
  mvm_backward(t, dD, B, dG, make_io(t.cfg.backward_io), t.k_bwd, t.seq_bwd, nullptr, false,
               nullptr);
  t.seq_bwd += (uint64_t)B;
  d2h_sync(t, G, dG, ng, pin ? pin + nd : nullptr);
}

int xb_tile_backward(xb_tile *h, const float *D, int B, float *G) {
  return guard([&] { backward_host(h, D, B, G); });
}

int xb_tile_backward_partial_dev(xb_tile *h, const float *dD, int B, const float *dAmaxD,
                                 float *dP) {
  return guard([&] {
    Tile &t = h->t;
    DevScope ds_(t.device);
    if (B < 0) raise("backward: batch must be >= 0");
    const xb_io_params &io = t.cfg.backward_io;
    if (io.bound_management != XB_BM_NONE)
      raise("backward_io.bound_management: not supported on row shards");
    IoDev d = make_io(io);
    // partials may run ahead of their finishes (chunked, overlapped
    // reductions): a partial's samples follow those still pending
    mvm_backward(t, dD, B, nullptr, d, t.k_bwd, t.seq_bwd + t.bwd_pending, dAmaxD, true, dP);
    t.bwd_pending += (uint64_t)B;
  });
}

int xb_tile_backward_finish_dev(xb_tile *h, const float *dPsum, int B, const float *dAmaxD,
                                float *dG) {
  return guard([&] {
    Tile &t = h->t;
    DevScope ds_(t.device);
    mvm_backward_finish(t, dPsum, B, dAmaxD, dG, make_io(t.cfg.backward_io), t.k_bwd, t.seq_bwd);
    t.seq_bwd += (uint64_t)B;
    t.bwd_pending -= std::min(t.bwd_pending, (uint64_t)B);
  });
}

int xb_rows_amax_dev(const float *dV, int B, int n, float *dOut, void *stream) {
  return guard([&] { launch_rows_amax(dV, B, n, n, dOut, (cudaStream_t)stream); });
}

int xb_tile_update_dev(xb_tile *h, const float *dX, const float *dD, int B, const double *lr,
                       const float *dAmaxD) {
  return guard([&] {
    Tile &t = h->t;
    DevScope ds_(t.device);
    if (B < 0) raise("update: batch must be >= 0");
    if (B == 0) return;
    check_lr_dev(lr, B, t.learning_rate);
    update_device(t, dX, dD, B, lr, dAmaxD, false, nullptr, nullptr, nullptr);
  });
}

int xb_tile_update(xb_tile *h, const float *X, const float *D, int B, const double *lr) {
  return guard([&] {
    Tile &t = h->t;
    DevScope ds_(t.device);
    if (B < 0) raise("update: batch must be >= 0");
    if (B == 0) return;
    float *dX = scratch_as<float>(t.s_y, (size_t)B * (t.C + t.R));
    float *dD = dX + (size_t)B * t.C;
    // small inputs: checked on the host before anything is enqueued
    const bool small =
        host_check_small({{X, (size_t)B * t.C, "update(x)"}, {D, (size_t)B * t.R, "update(d)"}});
    if (small) check_lr_host(X, D, B, t.C, t.R, lr, t.learning_rate);
    const size_t nx = (size_t)B * t.C, nd = (size_t)B * t.R;
    float *pin = io_stage(t, nx + nd);
    h2d(t, dX, X, nx, pin);
    h2d(t, dD, D, nd, pin ? pin + nx : nullptr);
    if (small) {
      update_device(t, dX, dD, B, lr, nullptr, false, nullptr, nullptr, nullptr);
      sync(t);
      return;
    }
    const std::initializer_list<Finite> in = {{dX, (size_t)B * t.C, "update(x)"},
                                              {dD, (size_t)B * t.R, "update(d)"}};
    try {
      check_lr_host(X, D, B, t.C, t.R, lr, t.learning_rate);
    } catch (...) { // check_input (tile.cpp:98-99) comes before translate's lr check
      check_finite_dev(t, in);
      throw;
    }
    // no host round trip before the launch: the update's x/d maxima kernel
    // also runs the finiteness test (bits 1, 2 of chk_dev, the order of
    // `in`), the pulse kernel reads the flag itself and leaves the tile
    // untouched if it is set; the host counters are rolled back and the
    // error raised after the sync
    clear_chk(t);
    const uint64_t seq_upd = t.seq_upd;
    const uint32_t calls = t.upd_calls;
    t.abort_flag = t.chk_dev;
    try {
      update_device(t, dX, dD, B, lr, nullptr, false, nullptr, nullptr, nullptr);
    } catch (...) {
      t.abort_flag = nullptr;
      throw;
    }
    t.abort_flag = nullptr;
    try {
      raise_if_nonfinite(t, in);
    } catch (...) {
      t.seq_upd = seq_upd;
      t.upd_calls = calls;
      throw;
    }
  });
}

int xb_tile_generate_trains(xb_tile *h, const float *X, const float *D, int B, const double *lr,
                            uint32_t *xw, uint32_t *dw, int32_t *bl) {
  return guard([&] {
    Tile &t = h->t;
    DevScope ds_(t.device);
    if (B <= 0) raise("generate_trains: batch must be >= 1");
    float *dX = scratch_as<float>(t.s_y, (size_t)B * (t.C + t.R));
    float *dD = dX + (size_t)B * t.C;
    XB_CUDA(cudaMemcpyAsync(dX, X, sizeof(float) * B * t.C, cudaMemcpyHostToDevice, t.stream));
    XB_CUDA(cudaMemcpyAsync(dD, D, sizeof(float) * B * t.R, cudaMemcpyHostToDevice, t.stream));
    check_finite_dev(t, {{dX, (size_t)B * t.C, "update(x)"}, {dD, (size_t)B * t.R, "update(d)"}});
    check_lr_host(X, D, B, t.C, t.R, lr, t.learning_rate);
    update_device(t, dX, dD, B, lr, nullptr, true, xw, dw, bl);
  });
}

int xb_tile_apply_trains(xb_tile *h, const uint32_t *xw, const uint32_t *dw, int B, int flip) {
  return guard([&] { // tile.cpp:158-169
    Tile &t = h->t;
    DevScope ds_(t.device);
    if (B < 0) raise("apply_trains: batch must be >= 0");
    if (B == 0) return;
    // reference-facing sample-major words -> internal layouts (x quads, d lines)
    const int ldb = train_ld(B);
    const size_t nx = (size_t)ldb * t.C, nd = (size_t)ldb * t.R;
    std::vector<uint32_t> hw(nx + nd, 0u);
    for (int b = 0; b < B; ++b) {
      for (int j = 0; j < t.C; ++j) hw[xq_index(j, b, t.C)] = xw[(size_t)b * t.C + j];
      for (int i = 0; i < t.R; ++i)
        hw[nx + (size_t)i * ldb + b] = dw[(size_t)b * t.R + i] ^ (flip ? 0x80000000u : 0u);
    }
    uint32_t *d = scratch_as<uint32_t>(t.s_params, nx + nd);
    XB_CUDA(cudaMemcpyAsync(d, hw.data(), (nx + nd) * 4, cudaMemcpyHostToDevice, t.stream));
    launch_pulse(t, d, d + nx, ldb, B, t.upd_calls);
    t.upd_calls += 1;
    t.seq_upd += (uint64_t)B;
    sync(t);
  });
}

int xb_tile_temporal_step(xb_tile *h, const xb_temporal_params *tp) { // tile.cpp:128-156
  return guard([&] {
    Tile &t = h->t;
    DevScope ds_(t.device);
    temporal_validate(*tp);
    if (!temporal_any(*tp)) return;
    ensure_xi(t);
    launch_temporal(t, *tp, t.temporal_calls++);
    wlo_reset(t);
    sync(t);
  });
}

int xb_tile_end_minibatch(xb_tile *h) { return xb_tile_temporal_step(h, &h->t.cfg.temporal); }

int xb_tile_attach_comm(xb_tile *h, xb_comm *c) {
  return guard([&] {
    Tile &t = h->t;
    Collective *col = comm_of(c);
    if (col && t.R == t.R_total && col->size() > 1)
      raise("attach_comm: the tile is not row-sharded (create it with an xb_shard)");
    if (col) col->bind(t.device);
    t.comm = col;
  });
}

int xb_tile_set_learning_rate(xb_tile *h, double lr) { // tile.cpp:121-126
  return guard([&] {
    if (!(lr > 0.0)) raise("learning_rate: must be > 0");
    h->t.learning_rate = lr;
  });
}

double xb_tile_learning_rate(const xb_tile *h) { return h->t.learning_rate; }

// ------------------------------------------------------------------ inference
static void model_validate(const xb_inference_model &m) { // inference.cpp:19-32
  if (!(m.t0 > 0.0)) raise("inference.t0: must be > 0");
  if (m.prog_noise_scale < 0.0 || m.read_noise_scale < 0.0 || m.nu_mean < 0.0 || m.nu_std < 0.0)
    raise("inference: noise scales and nu must be >= 0");
  if (m.nu_min < 0.0 || m.nu_max > 1.0 || m.nu_min > m.nu_max)
    raise("inference: nu clip must satisfy 0 <= nu_min <= nu_max <= 1");
  if (m.compensation_probes < 1) raise("inference.compensation_probes: must be >= 1");
}

int xb_tile_program(xb_tile *h, const float *target, const xb_inference_model *m, uint64_t seed) {
  return guard([&] { // inference.cpp:34-61
    Tile &t = h->t;
    DevScope ds_(t.device);
    model_validate(*m);
    const size_t n = (size_t)t.R * t.ld;
    if (!t.w0) {
      XB_CUDA(cudaMalloc(&t.w0, std::max<size_t>(n, 1) * sizeof(float)));
      XB_CUDA(cudaMalloc(&t.nu, std::max<size_t>(n, 1) * sizeof(float)));
    }
    float *dT = scratch_as<float>(t.s_y, (size_t)t.R * t.C);
    XB_CUDA(cudaMemcpyAsync(dT, target, sizeof(float) * (size_t)t.R * t.C, cudaMemcpyHostToDevice,
                            t.stream));
    launch_program(t, dT, *m, key_of(seed));
    wlo_reset(t);
    t.prog_t0 = m->t0;
    sync(t);
  });
}

int xb_tile_drift_to(xb_tile *h, double time_s) {
  return guard([&] { // inference.cpp:63-76
    Tile &t = h->t;
    DevScope ds_(t.device);
    if (!t.w0) raise("drift_to: tile has not been programmed");
    if (time_s < t.prog_t0) raise("drift_to: t < t0");
    launch_drift(t, time_s / t.prog_t0);
    wlo_reset(t);
    sync(t);
  });
}

int xb_tile_probe_readout(xb_tile *h, const xb_inference_model *m, double *out) {
  return guard([&] { // inference.cpp:85-95
    Tile &t = h->t;
    DevScope ds_(t.device);
    model_validate(*m);
    const int P = m->compensation_probes;
    std::vector<float> X((size_t)P * t.C, 1.0f), Y((size_t)P * t.R);
    forward_host(h, X.data(), P, Y.data(), noisy_io(t.cfg.forward_io, m->read_noise_scale));
    double acc = 0.0;
    for (int r = 0; r < P; ++r)
      for (int i = 0; i < t.R; ++i) acc += std::fabs((double)Y[(size_t)r * t.R + i]);
    *out = acc / P;
  });
}

int xb_tile_drift_compensation_factor(xb_tile *h, double baseline, const xb_inference_model *m,
                                      double *alpha) {
  double current = 0.0;
  int rc = xb_tile_probe_readout(h, m, &current);
  if (rc) return rc;
  return guard([&] { // inference.cpp:103-110
    if (current <= 1e-12) raise("drift_compensation_factor: degenerate readout (all-zero tile?)");
    *alpha = baseline / current;
  });
}

// ------------------------------------------------------------------ TransferTile
static void transfer_validate(const xb_transfer_config &s) { // compound.cpp:176-191
  if (s.transfer_every < 0) raise("transfer.transfer_every: must be >= 0 (0 disables transfer)");
  if (!(s.transfer_lr > 0.0)) raise("transfer.transfer_lr: must be > 0");
  if (s.columns_per_event < 1) raise("transfer.columns_per_event: must be >= 1");
  if (s.gamma < 0.0) raise("transfer.gamma: must be >= 0");
}

static xb_tile_config member_config(const xb_transfer_config &s, const xb_device_params &dev) {
  xb_tile_config c; // compound.cpp:31-42
  xb_default_config(&c);
  c.device = dev;
  c.forward_io = s.forward_io;
  c.backward_io = s.backward_io;
  c.update = s.update;
  c.temporal = s.temporal;
  c.mvm_precision = s.mvm_precision;
  return c;
}

int xb_transfer_create(const xb_transfer_config *cfg, int d_out, int d_in, uint64_t seed,
                       xb_transfer **out) {
  *out = nullptr;
  xb_tile_config fc = member_config(*cfg, cfg->fast_device);
  xb_tile_config sc = member_config(*cfg, cfg->slow_device);
  xb_tile *fast = nullptr, *slow = nullptr;
  int rc = xb_tile_create(&fc, d_out, d_in, derive_seed(seed, "fast"), nullptr, &fast);
  if (rc) return rc;
  rc = xb_tile_create(&sc, d_out, d_in, derive_seed(seed, "slow"), nullptr, &slow);
  if (rc) {
    xb_tile_destroy(fast);
    return rc;
  }
  rc = guard([&] { transfer_validate(*cfg); });
  if (rc) {
    xb_tile_destroy(fast);
    xb_tile_destroy(slow);
    return rc;
  }
  // both members on the fast tile's stream: the transfer's read (A) and
  // update (C) are ordered without events or host waits
  rc = xb_tile_set_stream(slow, fast->t.stream);
  if (rc) {
    xb_tile_destroy(fast);
    xb_tile_destroy(slow);
    return rc;
  }
  auto *t = new xb_transfer;
  t->cfg = *cfg;
  t->fast = fast;
  t->slow = slow;
  *out = t;
  return 0;
}

int xb_transfer_destroy(xb_transfer *t) {
  if (!t) return 0;
  xb_tile_destroy(t->slow); // borrows the fast tile's stream: first
  xb_tile_destroy(t->fast);
  t->onehot.release();
  t->readout.release();
  t->tmp.release();
  delete t;
  return 0;
}

static void mix_outputs(float *y, const float *ya, size_t n, double gamma) {
  for (size_t k = 0; k < n; ++k) y[k] = (float)((double)y[k] + gamma * (double)ya[k]);
}

int xb_transfer_forward(xb_transfer *t, const float *X, int B, float *Y) {
  return guard([&] { // compound.cpp:206-215
    forward_host(t->slow, X, B, Y, t->slow->t.cfg.forward_io);
    if (t->cfg.gamma != 0.0) {
      std::vector<float> ya((size_t)B * t->fast->t.R);
      forward_host(t->fast, X, B, ya.data(), t->fast->t.cfg.forward_io);
      mix_outputs(Y, ya.data(), ya.size(), t->cfg.gamma);
    }
  });
}

int xb_transfer_forward_noisy(xb_transfer *t, const float *X, int B, float *Y,
                              double extra_sigma) {
  return guard([&] { // compound.cpp:228-238
    forward_host(t->slow, X, B, Y, noisy_io(t->slow->t.cfg.forward_io, extra_sigma));
    if (t->cfg.gamma != 0.0) {
      std::vector<float> ya((size_t)B * t->fast->t.R);
      forward_host(t->fast, X, B, ya.data(), noisy_io(t->fast->t.cfg.forward_io, extra_sigma));
      mix_outputs(Y, ya.data(), ya.size(), t->cfg.gamma);
    }
  });
}

int xb_transfer_clone(const xb_transfer *t, xb_transfer **out) {
  *out = nullptr;
  xb_tile *fast = nullptr, *slow = nullptr; // compound.hpp:109-111: deep copy
  int rc = xb_tile_clone(t->fast, &fast);
  if (rc) return rc;
  rc = xb_tile_clone(t->slow, &slow);
  if (rc) {
    xb_tile_destroy(fast);
    return rc;
  }
  rc = xb_tile_set_stream(slow, fast->t.stream);
  if (rc) {
    xb_tile_destroy(slow);
    xb_tile_destroy(fast);
    return rc;
  }
  auto *c = new xb_transfer;
  c->cfg = t->cfg;
  c->fast = fast;
  c->slow = slow;
  c->counter = t->counter;
  c->events = t->events;
  c->next_column = t->next_column;
  *out = c;
  return 0;
}

int xb_transfer_backward(xb_transfer *t, const float *D, int B, float *G) {
  int rc = xb_tile_backward(t->slow, D, B, G); // compound.cpp:217-226
  if (rc || t->cfg.gamma == 0.0) return rc;
  std::vector<float> ga((size_t)B * t->fast->t.C);
  rc = xb_tile_backward(t->fast, D, B, ga.data());
  if (rc) return rc;
  mix_outputs(G, ga.data(), ga.size(), t->cfg.gamma);
  return 0;
}

// compound.cpp:257-267: a noisy read of A's column j (the forward of the
// one-hot e_j through the transfer io), then the pulsed update of C with x =
// e_j, d = readout.  All on the compound's one stream, nothing waits on the
// host: the read is a column gather plus the shared output stage
// (launch_column_read, bit-identical to the full forward), the update fires
// only the 32-column block holding j (x trains are zero elsewhere), and a
// zero readout is a no-op inside the update itself.  (Input noise or bound
// management on the transfer io take the full forward instead.)
static void transfer_step_impl(xb_transfer *tr) {
  Tile &a = tr->fast->t;
  Tile &c = tr->slow->t;
  const int j = tr->next_column;
  float *oh = scratch_as<float>(tr->onehot, a.C);
  float *ro = scratch_as<float>(tr->readout, a.R);
  const xb_io_params &iop = tr->cfg.has_transfer_io ? tr->cfg.transfer_io : tr->cfg.forward_io;
  io_validate(iop, "transfer_io");
  const IoDev io = make_io(iop);
  if (io.sigma_inp > 0.0 || io.bm) {
    std::vector<float> e(a.C, 0.f);
    e[j] = 1.0f;
    XB_CUDA(cudaMemcpyAsync(oh, e.data(), sizeof(float) * a.C, cudaMemcpyHostToDevice, a.stream));
    XB_CUDA(cudaStreamSynchronize(a.stream)); // e is a host temporary
    forward_device(a, oh, 1, ro, iop);
  } else {
    launch_column_read(a, j, io, a.k_fwd, a.seq_fwd, ro, oh);
    a.seq_fwd += 1;
  }
  const double lr = tr->cfg.transfer_lr;
  update_device(c, oh, ro, 1, &lr, nullptr, false, nullptr, nullptr, nullptr, j);
  tr->next_column = (j + 1) % a.C;
}

static void tick(xb_transfer *t) { // compound.cpp:247-255
  ++t->counter;
  if (t->cfg.transfer_every > 0 && t->counter % t->cfg.transfer_every == 0) {
    ++t->events;
    for (int n = 0; n < t->cfg.columns_per_event; ++n) transfer_step_impl(t);
  }
}

int xb_transfer_step(xb_transfer *t) {
  return guard([&] { transfer_step_impl(t); });
}

int xb_transfer_update(xb_transfer *t, const float *X, const float *D, int B, const double *lr) {
  return guard([&] { // compound.cpp:240-245
    Tile &a = t->fast->t;
    if (t->cfg.units_in_mbatch || t->cfg.transfer_every == 0) {
      if (xb_tile_update(t->fast, X, D, B, lr)) raise(g_err);
      if (!t->cfg.units_in_mbatch)
        for (int b = 0; b < B; ++b) tick(t);
      return;
    }
    // ticks interleave with samples: split the batch at every transfer event
    int b = 0;
    while (b < B) {
      const long to_event = t->cfg.transfer_every - (t->counter % t->cfg.transfer_every);
      const int n = (int)std::min<long>(to_event, B - b);
      if (xb_tile_update(t->fast, X + (size_t)b * a.C, D + (size_t)b * a.R, n, lr ? lr + b : nullptr))
        raise(g_err);
      for (int k = 0; k < n; ++k) tick(t);
      b += n;
    }
  });
}

int xb_transfer_end_minibatch(xb_transfer *t) {
  return guard([&] { // compound.cpp:287-293
    if (t->cfg.units_in_mbatch) tick(t);
    if (xb_tile_end_minibatch(t->fast)) raise(g_err);
    if (xb_tile_end_minibatch(t->slow)) raise(g_err);
  });
}

int xb_transfer_get_weights(const xb_transfer *t, float *w) {
  return guard([&] { // compound.cpp:269-280
    if (xb_tile_get_weights(t->slow, w)) raise(g_err);
    if (t->cfg.gamma != 0.0) {
      std::vector<float> a((size_t)t->fast->t.R * t->fast->t.C);
      if (xb_tile_get_weights(t->fast, a.data())) raise(g_err);
      mix_outputs(w, a.data(), a.size(), t->cfg.gamma);
    }
  });
}

int xb_transfer_set_weights(xb_transfer *t, const float *w) {
  return guard([&] { // compound.cpp:282-285
    if (xb_tile_set_weights(t->slow, w)) raise(g_err);
    std::vector<float> z((size_t)t->fast->t.R * t->fast->t.C, 0.f);
    if (xb_tile_set_weights(t->fast, z.data())) raise(g_err);
  });
}

long xb_transfer_events(const xb_transfer *t) { return t->events; }
xb_tile *xb_transfer_fast(xb_transfer *t) { return t->fast; }
xb_tile *xb_transfer_slow(xb_transfer *t) { return t->slow; }


} // extern "C"

// ============================================================== UnitCellTile
namespace xb {

static xb_tile_config uc_member_config(const xb_unitcell_config &c, const xb_device_params &d) {
  xb_tile_config m; // compound.cpp:31-42
  xb_default_config(&m);
  m.device = d;
  m.forward_io = c.forward_io;
  m.backward_io = c.backward_io;
  m.update = c.update;
  m.temporal = c.temporal;
  m.mvm_precision = c.mvm_precision;
  return m;
}

static void unitcell_validate(const xb_unitcell_config &c) { // compound.cpp:12-27
  if (c.n_devices < 1) raise("unit_cell.devices: need at least one device");
  if (c.n_devices > XB_MAX_CELL_DEVICES) raise("unit_cell.gains: length must match devices");
  for (int k = 0; k < c.n_devices; ++k)
    if (!std::isfinite(c.gains[k])) raise("unit_cell.gains: entries must be finite");
  for (int k = 0; k < c.n_devices; ++k)
    device_validate(c.devices[k], ("unit_cell.devices[" + std::to_string(k) + "]").c_str());
}

// the compound's handle: W_eff only (no device arrays), keys from the compound
// seed, so its "forward"/"backward"/"update" streams are the compound's own
static xb_tile *view_tile_create(const xb_tile_config &cfg, int R, int C, uint64_t seed) {
  auto h = std::make_unique<xb_tile>();
  Tile &t = h->t;
  DevScope ds_(t.device);
  t.cfg = cfg;
  t.R = R;
  t.C = C;
  t.R_total = R;
  t.ld = (int)ld_of(C);
  tile_init_keys(t, seed);
  XB_CUDA(cudaStreamCreateWithFlags(&t.stream, cudaStreamNonBlocking));
  t.own_stream = true;
  const size_t n = (size_t)R * t.ld;
  XB_CUDA(cudaMalloc(&t.W, std::max<size_t>(n, 1) * sizeof(float)));
  XB_CUDA(cudaMemsetAsync(t.W, 0, n * sizeof(float), t.stream));
  return h.release();
}

static void uc_share_stream(xb_unitcell *u) {
  for (xb_tile *m : u->members) {
    if (m->t.own_stream && m->t.stream) {
      XB_CUDA(cudaStreamSynchronize(m->t.stream));
      cudaStreamDestroy(m->t.stream);
    }
    m->t.own_stream = false;
    m->t.stream = u->eff->t.stream;
  }
}

static void uc_effective(xb_unitcell *u) {
  if (!u->dirty) return;
  const float *w[XB_MAX_CELL_DEVICES];
  for (size_t k = 0; k < u->members.size(); ++k) w[k] = u->members[k]->t.W;
  Tile &e = u->eff->t;
  launch_effective(e.W, w, u->cfg.gains, (int)u->members.size(), e.R, e.C, e.ld, e.stream);
  u->dirty = false;
}

static void uc_free(xb_unitcell *u) {
  for (xb_tile *m : u->members) xb_tile_destroy(m);
  if (u->eff) xb_tile_destroy(u->eff);
  delete u;
}

// compound.cpp:109-147 for B samples in order: one translate + trains per
// sample on the compound's update stream (grain per sample), then each member
// fires the trains of its samples in one weight-stationary pulse launch
static void uc_update(xb_unitcell *u, const float *X, const float *D, int B, const double *lr) {
  Tile &e = u->eff->t;
  const int K = (int)u->members.size();
  const bool rr = u->cfg.policy == XB_UC_ROUND_ROBIN;
  double grain_all = 0.0;
  for (int k = 0; k < K; ++k) grain_all += std::fabs(u->cfg.gains[k]) * u->cfg.devices[k].dw_min;
  std::vector<double> lre(B, 0.0);
  std::vector<double> grain(B, 0.0);
  std::vector<int> member(B, -1);
  int cursor = u->next_member;
  bool any = false;
  for (int b = 0; b < B; ++b) {
    const double l = lr ? lr[b] : e.learning_rate;
    bool xz = true, dz = true;
    for (int j = 0; j < e.C && xz; ++j) xz = X[(size_t)b * e.C + j] == 0.f;
    for (int i = 0; i < e.R && dz; ++i) dz = D[(size_t)b * e.R + i] == 0.f;
    if (l == 0.0 || xz || dz) continue; // :113-115, no draw, cursor unchanged
    double g = grain_all;
    if (rr) {
      member[b] = cursor;
      g = std::fabs(u->cfg.gains[cursor]) * u->cfg.devices[cursor].dw_min;
      cursor = (cursor + 1) % K;
    }
    if (g == 0.0) continue; // zero-gain member (or all gains zero): a no-op event
    if (!(l > 0.0)) raise("translate: learning rate must be > 0"); // pulsed.cpp:27-29
    lre[b] = l;
    grain[b] = g;
    any = true;
  }
  u->next_member = cursor;
  if (!any) return;
  u->dirty = true;
  const int ldb = train_ld(B);
  UpdBufs ub = upd_bufs(e, B, false);
  float *dX = scratch_as<float>(e.s_y, (size_t)B * (e.C + e.R));
  float *dD = dX + (size_t)B * e.C;
  char *aux = (char *)e.s_params.get((size_t)B * (sizeof(double) + sizeof(int)) + 256);
  double *dG = (double *)aux;
  int *dIdx = (int *)(aux + (size_t)B * sizeof(double));
  XB_CUDA(cudaMemcpyAsync(dX, X, sizeof(float) * B * e.C, cudaMemcpyHostToDevice, e.stream));
  XB_CUDA(cudaMemcpyAsync(dD, D, sizeof(float) * B * e.R, cudaMemcpyHostToDevice, e.stream));
  XB_CUDA(cudaMemcpyAsync(ub.lr, lre.data(), sizeof(double) * B, cudaMemcpyHostToDevice, e.stream));
  XB_CUDA(cudaMemcpyAsync(dG, grain.data(), sizeof(double) * B, cudaMemcpyHostToDevice,
                          e.stream));
  launch_rows_amax2(dX, e.C, ub.xm, dD, e.R, ub.dm, B, e.stream);
  launch_trains(e, dX, dD, B, ub.lr, 0.0, ub.xm, ub.dm, e.seq_upd, ub.xw, ub.dw, ldb, ub.bl,
                nullptr, nullptr, false, dG);
  e.seq_upd += (uint64_t)B;
  if (!rr) {
    for (int k = 0; k < K; ++k) {
      if (u->cfg.gains[k] == 0.0) continue;
      Tile &m = u->members[k]->t;
      launch_pulse(m, ub.xw, ub.dw, ldb, B, m.upd_calls++, u->cfg.gains[k] < 0.0);
    }
  } else {
    std::vector<int> idx;
    idx.reserve(B);
    uint32_t *gx = scratch_as<uint32_t>(e.s_io, (size_t)ldb * (e.C + e.R));
    for (int k = 0; k < K; ++k) {
      idx.clear();
      for (int b = 0; b < B; ++b)
        if (member[b] == k && lre[b] != 0.f) idx.push_back(b);
      if (idx.empty()) continue;
      const int n = (int)idx.size(), ldn = train_ld(n);
      XB_CUDA(cudaMemcpyAsync(dIdx, idx.data(), sizeof(int) * n, cudaMemcpyHostToDevice,
                              e.stream));
      launch_gather_samples(ub.xw, ldb, e.C, dIdx, n, gx, ldn, e.stream, true);
      launch_gather_samples(ub.dw, ldb, e.R, dIdx, n, gx + (size_t)ldn * e.C, ldn, e.stream);
      Tile &m = u->members[k]->t;
      launch_pulse(m, gx, gx + (size_t)ldn * e.C, ldn, n, m.upd_calls++, u->cfg.gains[k] < 0.0);
      sync(e); // idx / gather buffers are reused by the next member
    }
  }
  sync(e);
}

} // namespace xb

extern "C" {

void xb_default_unitcell_config(xb_unitcell_config *c) { // compound.hpp:15-28
  std::memset(c, 0, sizeof *c);
  c->n_devices = 1;
  xb_default_device(&c->devices[0]);
  c->gains[0] = 1.0;
  c->policy = XB_UC_ALL_TOGETHER;
  xb_default_io(&c->forward_io);
  xb_default_io(&c->backward_io);
  c->update = xb_update_params{31, 0, XB_PULSE_STOCHASTIC};
  c->mvm_precision = XB_MVM_TF32X3;
}

int xb_unitcell_create(const xb_unitcell_config *cfg, int d_out, int d_in, uint64_t seed,
                       xb_unitcell **out) {
  *out = nullptr;
  auto *u = new xb_unitcell;
  u->cfg = *cfg;
  int rc = guard([&] { unitcell_validate(*cfg); });
  for (int k = 0; rc == 0 && k < cfg->n_devices; ++k) { // compound.cpp:52-64
    const xb_tile_config mc = uc_member_config(*cfg, cfg->devices[k]);
    xb_tile *m = nullptr;
    rc = xb_tile_create(&mc, d_out, d_in,
                        k == 0 ? seed : derive_seed_idx(seed, "cell_member", (uint64_t)k), nullptr,
                        &m);
    if (rc == 0) u->members.push_back(m);
  }
  if (rc == 0)
    rc = guard([&] {
      u->eff = view_tile_create(uc_member_config(*cfg, cfg->devices[0]), d_out, d_in, seed);
      uc_share_stream(u);
    });
  if (rc) {
    uc_free(u);
    return rc;
  }
  *out = u;
  return 0;
}

int xb_unitcell_destroy(xb_unitcell *u) {
  if (u) uc_free(u);
  return 0;
}

int xb_unitcell_clone(const xb_unitcell *src, xb_unitcell **out) {
  *out = nullptr;
  auto *u = new xb_unitcell;
  u->cfg = src->cfg;
  u->dirty = src->dirty;
  u->next_member = src->next_member;
  int rc = 0;
  for (xb_tile *m : src->members) {
    xb_tile *c = nullptr;
    if ((rc = xb_tile_clone(m, &c))) break;
    u->members.push_back(c);
  }
  if (rc == 0)
    rc = guard([&] {
      const Tile &s = src->eff->t;
      XB_CUDA(cudaStreamSynchronize(s.stream));
      u->eff = view_tile_create(s.cfg, s.R, s.C, s.seed);
      Tile &t = u->eff->t;
      t.seq_fwd = s.seq_fwd;
      t.seq_bwd = s.seq_bwd;
      t.seq_upd = s.seq_upd;
      t.learning_rate = s.learning_rate;
      XB_CUDA(cudaMemcpyAsync(t.W, s.W, (size_t)t.R * t.ld * sizeof(float),
                              cudaMemcpyDeviceToDevice, t.stream));
      uc_share_stream(u);
      sync(t);
    });
  if (rc) {
    uc_free(u);
    return rc;
  }
  *out = u;
  return 0;
}

int xb_unitcell_forward(xb_unitcell *u, const float *X, int B, float *Y) {
  return guard([&] { // compound.cpp:82-88
    uc_effective(u);
    forward_host(u->eff, X, B, Y, u->cfg.forward_io, false);
  });
}

int xb_unitcell_forward_noisy(xb_unitcell *u, const float *X, int B, float *Y,
                              double extra_sigma) {
  return guard([&] { // compound.cpp:98-107
    uc_effective(u);
    forward_host(u->eff, X, B, Y, noisy_io(u->cfg.forward_io, extra_sigma), false);
  });
}

int xb_unitcell_backward(xb_unitcell *u, const float *D, int B, float *G) {
  return guard([&] { // compound.cpp:90-96
    uc_effective(u);
    backward_host(u->eff, D, B, G, false);
  });
}

int xb_unitcell_update(xb_unitcell *u, const float *X, const float *D, int B, const double *lr) {
  return guard([&] {
    if (B < 0) raise("update: batch must be >= 0");
    if (B > 0) uc_update(u, X, D, B, lr);
  });
}

int xb_unitcell_get_weights(xb_unitcell *u, float *w) {
  return guard([&] { // compound.cpp:149
    uc_effective(u);
    if (xb_tile_get_weights(u->eff, w)) raise(g_err);
  });
}

int xb_unitcell_set_weights(xb_unitcell *u, const float *w) {
  return guard([&] { // compound.cpp:151-167
    const double g0 = u->cfg.gains[0];
    if (g0 == 0.0) raise("set_weights: unit cell with zero first gain cannot be programmed");
    const Tile &e = u->eff->t;
    const size_t n = (size_t)e.R * e.C;
    std::vector<float> scaled(n);
    for (size_t c = 0; c < n; ++c) scaled[c] = (float)((double)w[c] / g0);
    if (xb_tile_set_weights(u->members[0], scaled.data())) raise(g_err);
    std::fill(scaled.begin(), scaled.end(), 0.f);
    for (size_t k = 1; k < u->members.size(); ++k)
      if (xb_tile_set_weights(u->members[k], scaled.data())) raise(g_err);
    u->dirty = true;
  });
}

int xb_unitcell_end_minibatch(xb_unitcell *u) {
  return guard([&] { // compound.cpp:169-174
    for (xb_tile *m : u->members)
      if (xb_tile_end_minibatch(m)) raise(g_err);
    u->dirty = true;
  });
}

int xb_unitcell_n_members(const xb_unitcell *u) { return (int)u->members.size(); }

xb_tile *xb_unitcell_member(xb_unitcell *u, int k) {
  return (k >= 0 && k < (int)u->members.size()) ? u->members[k] : nullptr;
}

} // extern "C"
