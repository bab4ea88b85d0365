// xbarsim_b200/tile.hpp -- the reference's C++ tile API over the B200 C ABI.
//
// Header-only host layer mirroring proj/include/xbarsim/{tile,compound,
// inference,device,io,pulsed}.hpp: the same class names, settings structs
// (same fields, same defaults), virtual surface and error behaviour, so a
// caller of xbarsim::AnalogTile / TransferTile switches by changing the
// namespace.  All compute goes through libxbtile.so (include/xbtile.h); link
// with -lxbtile.
//
// Batching bridge: update() validates its arguments eagerly
// (length, finiteness, lr; proj/src/tile.cpp:65-75,97-101,
// proj/src/pulsed.cpp:27-29) and queues the sample; the queue is applied as
// ONE weight-stationary batched update (samples in order) before the next
// forward/backward/get_weights/set_weights/end_minibatch/clone, which is
// exactly equivalent because the reference NN host applies all updates of a
// mini-batch after all its forwards/backwards (proj/src/nn.cpp:708-735).
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <limits>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <tuple>
#include <utility>
#include <vector>

#include "../xbtile.h"

namespace xbarsim_b200 {

// proj/include/xbarsim/common.hpp:15-18
class Error : public std::runtime_error {
public:
  explicit Error(const std::string &msg) : std::runtime_error(msg) {}
};

inline void check(int rc) {
  if (rc != 0) throw Error(xb_last_error());
}

enum class DeviceKind { constant_step = XB_CONSTANT_STEP, linear_step = XB_LINEAR_STEP,
                        soft_bounds = XB_SOFT_BOUNDS, exp_step = XB_EXP_STEP };
enum class NoiseManagement { none = XB_NM_NONE, abs_max = XB_NM_ABS_MAX };
enum class PulseType { stochastic = XB_PULSE_STOCHASTIC,
                       deterministic_implicit = XB_PULSE_DETERMINISTIC };
enum class BoundManagement { none = XB_BM_NONE, iterative = XB_BM_ITERATIVE };
enum class MvmPrecision { fp32 = XB_MVM_FP32, tf32 = XB_MVM_TF32, tf32x3 = XB_MVM_TF32X3 };
enum class WeightPrecision { automatic = XB_W_AUTO, fp32 = XB_W_FP32, fp32x2 = XB_W_FP32X2 };

// proj/include/xbarsim/device.hpp:24-39
struct DeviceParams {
  DeviceKind kind = DeviceKind::constant_step;
  double dw_min = 0.001;
  double dw_min_dtod = 0.0;
  double dw_min_std = 0.0;
  double up_down = 0.0;
  double up_down_dtod = 0.0;
  double w_max = 1.0;
  double w_min = -1.0;
  double w_max_dtod = 0.0;
  double w_min_dtod = 0.0;
  double slope = 1.0;
  double gamma = 2.0;
};

// proj/include/xbarsim/io.hpp:21-33 (+ additive bound management)
struct IOParams {
  int dac_bits = 7;
  int adc_bits = 9;
  double input_bound = 1.0;
  double output_bound = 12.0;
  double sigma_inp = 0.0;
  double sigma_out = 0.06;
  double sigma_w = 0.0;
  NoiseManagement noise_management = NoiseManagement::abs_max;
  bool is_perfect = false;
  BoundManagement bound_management = BoundManagement::none;
  int bm_max_iter = 10;
};

// proj/include/xbarsim/pulsed.hpp:21-27
struct UpdateParams {
  int bl = 31;
  bool bl_management = false;
  PulseType pulse_type = PulseType::stochastic;
};

// proj/include/xbarsim/pulsed.hpp:37-50: Bernoulli pulse trains, slot-major
struct PulseTrains {
  int bl = 0;
  int x_lines = 0;
  int d_lines = 0;
  std::vector<uint8_t> x_bits, d_bits;

  bool x_bit(int slot, int line) const {
    return x_bits[static_cast<size_t>(slot) * x_lines + line] != 0;
  }
  bool d_bit(int slot, int line) const {
    return d_bits[static_cast<size_t>(slot) * d_lines + line] != 0;
  }
};

// proj/include/xbarsim/tile.hpp:24-36
struct TemporalParams {
  double decay_rate = 0.0;
  double decay_dtod = 0.0;
  double diffusion_sigma = 0.0;
  double diffusion_dtod = 0.0;
  double reset_prob = 0.0;
  double reset_dtod = 0.0;
  bool any() const { return decay_rate > 0.0 || diffusion_sigma > 0.0 || reset_prob > 0.0; }
};

// proj/include/xbarsim/tile.hpp:38-44 (+ additive precision mode)
struct TileSettings {
  DeviceParams device;
  IOParams forward_io;
  IOParams backward_io;
  UpdateParams update;
  TemporalParams temporal;
  MvmPrecision mvm_precision = MvmPrecision::tf32x3;
  WeightPrecision weight_precision = WeightPrecision::automatic;
};

// proj/include/xbarsim/compound.hpp:76-91
struct TransferSettings {
  DeviceParams fast_device;
  DeviceParams slow_device;
  IOParams forward_io;
  IOParams backward_io;
  UpdateParams update;
  TemporalParams temporal;
  int transfer_every = 1;
  bool units_in_mbatch = false;
  double transfer_lr = 0.1;
  int columns_per_event = 1;
  double gamma = 0.0;
  bool has_transfer_io = false;
  IOParams transfer_io;
  MvmPrecision mvm_precision = MvmPrecision::tf32x3;
};

// proj/include/xbarsim/inference.hpp:21-36
struct InferenceNoiseModel {
  double prog_noise_scale = 1.0;
  double prog_c0 = 0.26;
  double prog_c1 = 1.66;
  double prog_c2 = 0.33;
  double read_noise_scale = 0.0;
  double nu_mean = 0.06;
  double nu_std = 0.03;
  double t0 = 20.0;
  double nu_min = 0.0;
  double nu_max = 1.0;
  int compensation_probes = 10;
  double prog_sigma(double w) const {
    const double a = std::fabs(w);
    return prog_noise_scale * (prog_c0 + prog_c1 * a + prog_c2 * a * a);
  }
};

// proj/include/xbarsim/matrix.hpp:18-50 (row-major doubles)
class Matrix {
public:
  Matrix() = default;
  Matrix(int rows, int cols, double fill = 0.0)
      : rows_(rows), cols_(cols), data_(static_cast<size_t>(rows) * cols, fill) {}
  int rows() const { return rows_; }
  int cols() const { return cols_; }
  size_t size() const { return data_.size(); }
  double &operator()(int i, int j) { return data_[static_cast<size_t>(i) * cols_ + j]; }
  double operator()(int i, int j) const { return data_[static_cast<size_t>(i) * cols_ + j]; }
  double *data() { return data_.data(); }
  const double *data() const { return data_.data(); }
  bool same_shape(const Matrix &o) const { return rows_ == o.rows_ && cols_ == o.cols_; }
  bool operator==(const Matrix &o) const {
    return rows_ == o.rows_ && cols_ == o.cols_ && data_ == o.data_;
  }

private:
  int rows_ = 0, cols_ = 0;
  std::vector<double> data_;
};

// proj/include/xbarsim/device.hpp:41-49: per-crosspoint sampled parameters
struct DeviceRealization {
  double dw_min_up = 0.0;
  double dw_min_down = 0.0;
  double w_max = 0.0;
  double w_min = 0.0;
  double slope = 0.0;
  double gamma = 0.0;
};

// proj/include/xbarsim/device.hpp:58-79: host snapshot of the realized device
// array (the B200 tile keeps it in HBM as fp32 SoA; device() downloads it)
class DeviceMatrix {
public:
  DeviceMatrix() = default;
  DeviceMatrix(const DeviceParams &params, int rows, int cols)
      : params_(params), rows_(rows), cols_(cols), cells_(static_cast<size_t>(rows) * cols) {}
  int rows() const { return rows_; }
  int cols() const { return cols_; }
  const DeviceParams &params() const { return params_; }
  const DeviceRealization &at(int i, int j) const {
    return cells_[static_cast<size_t>(i) * cols_ + j];
  }
  DeviceRealization &at(int i, int j) { return cells_[static_cast<size_t>(i) * cols_ + j]; }
  // proj/src/device.cpp:79-88: clip to the cell's own bounds
  double clip(int i, int j, double w) const {
    const DeviceRealization &c = at(i, j);
    return std::fmin(std::fmax(w, c.w_min), c.w_max);
  }

private:
  DeviceParams params_;
  int rows_ = 0, cols_ = 0;
  std::vector<DeviceRealization> cells_;
};

namespace detail {
inline xb_device_params to_c(const DeviceParams &p) {
  xb_device_params d;
  xb_default_device(&d);
  d.kind = static_cast<int32_t>(p.kind);
  d.dw_min = p.dw_min;
  d.dw_min_dtod = p.dw_min_dtod;
  d.dw_min_std = p.dw_min_std;
  d.up_down = p.up_down;
  d.up_down_dtod = p.up_down_dtod;
  d.w_max = p.w_max;
  d.w_min = p.w_min;
  d.w_max_dtod = p.w_max_dtod;
  d.w_min_dtod = p.w_min_dtod;
  d.slope = p.slope;
  d.gamma = p.gamma;
  return d;
}
inline DeviceParams from_c(const xb_device_params &d) {
  DeviceParams p;
  p.kind = static_cast<DeviceKind>(d.kind);
  p.dw_min = d.dw_min;
  p.dw_min_dtod = d.dw_min_dtod;
  p.dw_min_std = d.dw_min_std;
  p.up_down = d.up_down;
  p.up_down_dtod = d.up_down_dtod;
  p.w_max = d.w_max;
  p.w_min = d.w_min;
  p.w_max_dtod = d.w_max_dtod;
  p.w_min_dtod = d.w_min_dtod;
  p.slope = d.slope;
  p.gamma = d.gamma;
  return p;
}
inline xb_io_params to_c(const IOParams &p) {
  xb_io_params d;
  xb_default_io(&d);
  d.dac_bits = p.dac_bits;
  d.adc_bits = p.adc_bits;
  d.input_bound = p.input_bound;
  d.output_bound = p.output_bound;
  d.sigma_inp = p.sigma_inp;
  d.sigma_out = p.sigma_out;
  d.sigma_w = p.sigma_w;
  d.noise_management = static_cast<int32_t>(p.noise_management);
  d.is_perfect = p.is_perfect ? 1 : 0;
  d.bound_management = static_cast<int32_t>(p.bound_management);
  d.bm_max_iter = p.bm_max_iter;
  return d;
}
inline xb_update_params to_c(const UpdateParams &p) {
  return xb_update_params{p.bl, p.bl_management ? 1 : 0, static_cast<int32_t>(p.pulse_type)};
}
inline xb_temporal_params to_c(const TemporalParams &p) {
  return xb_temporal_params{p.decay_rate,     p.decay_dtod, p.diffusion_sigma,
                            p.diffusion_dtod, p.reset_prob, p.reset_dtod};
}
inline xb_tile_config to_c(const TileSettings &s) {
  xb_tile_config c;
  xb_default_config(&c);
  c.device = to_c(s.device);
  c.forward_io = to_c(s.forward_io);
  c.backward_io = to_c(s.backward_io);
  c.update = to_c(s.update);
  c.temporal = to_c(s.temporal);
  c.mvm_precision = static_cast<int32_t>(s.mvm_precision);
  c.weight_precision = static_cast<int32_t>(s.weight_precision);
  return c;
}
inline xb_inference_model to_c(const InferenceNoiseModel &m) {
  xb_inference_model r;
  xb_default_inference_model(&r);
  r.prog_noise_scale = m.prog_noise_scale;
  r.prog_c0 = m.prog_c0;
  r.prog_c1 = m.prog_c1;
  r.prog_c2 = m.prog_c2;
  r.read_noise_scale = m.read_noise_scale;
  r.nu_mean = m.nu_mean;
  r.nu_std = m.nu_std;
  r.t0 = m.t0;
  r.nu_min = m.nu_min;
  r.nu_max = m.nu_max;
  r.compensation_probes = m.compensation_probes;
  return r;
}
inline std::vector<float> to_f(std::span<const double> v) {
  return std::vector<float>(v.begin(), v.end());
}
inline std::vector<double> to_d(const std::vector<float> &v) {
  return std::vector<double>(v.begin(), v.end());
}
// proj/src/tile.cpp:65-75
inline void check_input(std::span<const double> v, int expected, const char *what) {
  if (static_cast<int>(v.size()) != expected)
    throw Error(std::string(what) + ": length " + std::to_string(v.size()) + ", expected " +
                std::to_string(expected));
  for (double x : v)
    if (!std::isfinite(x)) throw Error(std::string(what) + ": non-finite entry");
}
// One pass over an update vector: check_input's length and finiteness (raised
// at once, in the reference's order), and whether it is all zero or leaves
// the fp32 range (raised by the caller after the reference's earlier checks).
struct UpdateScan {
  bool zero = true, beyond_f32 = false;
};
inline UpdateScan scan_update_input(std::span<const double> v, int expected, const char *what) {
  if (static_cast<int>(v.size()) != expected)
    throw Error(std::string(what) + ": length " + std::to_string(v.size()) + ", expected " +
                std::to_string(expected));
  constexpr double fmax = static_cast<double>(std::numeric_limits<float>::max());
  bool bad = false, zero = true, big = false;
  for (double x : v) {
    const double a = std::fabs(x);
    bad |= !(a <= std::numeric_limits<double>::max()); // Inf or NaN
    zero &= x == 0.0;
    big |= a > fmax;
  }
  if (bad) throw Error(std::string(what) + ": non-finite entry");
  return {zero, big};
}
} // namespace detail

// proj/src/device.cpp:100-132
inline DeviceParams device_preset(std::string_view name) {
  xb_device_params p;
  check(xb_device_preset(std::string(name).c_str(), &p));
  return detail::from_c(p);
}

// proj/src/io.cpp:32-40
inline IOParams perfect_io() {
  IOParams io;
  io.is_perfect = true;
  io.dac_bits = 0;
  io.adc_bits = 0;
  io.sigma_out = 0.0;
  io.noise_management = NoiseManagement::none;
  return io;
}

// proj/include/xbarsim/tile.hpp:47-70
class TileBase {
public:
  virtual ~TileBase() = default;
  virtual int d_out() const = 0;
  virtual int d_in() const = 0;
  virtual std::vector<double> forward(std::span<const double> x) = 0;
  virtual std::vector<double> backward(std::span<const double> d) = 0;
  virtual void update(std::span<const double> x, std::span<const double> d, double lr) = 0;
  virtual std::vector<double> forward_noisy(std::span<const double> x,
                                            double extra_weight_sigma) = 0;
  virtual Matrix get_weights() const = 0;
  virtual void set_weights(const Matrix &w) = 0;
  virtual void end_minibatch() = 0;
  virtual std::unique_ptr<TileBase> clone() const = 0;

  // batched extras of the B200 path: B samples per call,
  // row-major fp32 host buffers; each equals B sequential reference calls on
  // stationary weights.  lr[B] may be null (the tile's learning rate).
  virtual void forward_batch(const float *X, int B, float *Y) = 0;
  virtual void forward_noisy_batch(const float *X, int B, float *Y, double extra_sigma) = 0;
  virtual void backward_batch(const float *D, int B, float *G) = 0;
  virtual void update_batch(const float *X, const float *D, int B, const double *lr) = 0;
};

// proj/include/xbarsim/tile.hpp:75-131, on the GPU
class AnalogTile : public TileBase {
public:
  AnalogTile(int d_out, int d_in, const TileSettings &settings, uint64_t seed)
      : settings_(settings) {
    const xb_tile_config c = detail::to_c(settings);
    check(xb_tile_create(&c, d_out, d_in, seed, nullptr, &h_));
    d_out_ = d_out;
    d_in_ = d_in;
  }
  ~AnalogTile() override {
    if (h_ && owned_) xb_tile_destroy(h_);
  }
  // borrowed view of a member tile owned by a compound (not destroyed here)
  AnalogTile(xb_tile *borrowed, int d_out, int d_in, const TileSettings &settings)
      : settings_(settings), h_(borrowed), d_out_(d_out), d_in_(d_in), owned_(false) {}
  AnalogTile(const AnalogTile &o) : settings_(o.settings_), d_out_(o.d_out_), d_in_(o.d_in_) {
    // proj/include/xbarsim/tile.hpp:91: clone = deep copy (queued updates applied first)
    o.flush();
    check(xb_tile_clone(o.h_, &h_));
  }
  AnalogTile &operator=(const AnalogTile &) = delete;

  int d_out() const override { return d_out_; }
  int d_in() const override { return d_in_; }

  std::vector<double> forward(std::span<const double> x) override {
    detail::check_input(x, d_in_, "forward");
    flush();
    auto xf = detail::to_f(x);
    std::vector<float> y(d_out_);
    check(xb_tile_forward(h_, xf.data(), 1, y.data()));
    return detail::to_d(y);
  }
  std::vector<double> backward(std::span<const double> d) override {
    detail::check_input(d, d_out_, "backward");
    flush();
    auto df = detail::to_f(d);
    std::vector<float> g(d_in_);
    check(xb_tile_backward(h_, df.data(), 1, g.data()));
    return detail::to_d(g);
  }
  // proj/src/tile.cpp:97-101 via the batching bridge
  void update(std::span<const double> x, std::span<const double> d, double lr) override {
    // (one scan per vector for every check below, then the fp32 append: the
    // per-sample update is host-bound)
    const detail::UpdateScan sx = detail::scan_update_input(x, d_in_, "update(x)");
    const detail::UpdateScan sd = detail::scan_update_input(d, d_out_, "update(d)");
    if (lr == 0.0 || sx.zero || sd.zero) return; // proj/src/pulsed.cpp:122-124, no draw
    if (!(lr > 0.0)) throw Error("translate: learning rate must be > 0");
    // the queue stores fp32 x/d (the device arithmetic); a finite double
    // beyond the fp32 range would become Inf there, so it is rejected here,
    // at the call, like check_input's non-finite entries
    if (sx.beyond_f32)
      throw Error("update(x): entry exceeds the fp32 range of the B200 tile");
    if (sd.beyond_f32)
      throw Error("update(d): entry exceeds the fp32 range of the B200 tile");
    qx_.insert(qx_.end(), x.begin(), x.end());
    qd_.insert(qd_.end(), d.begin(), d.end());
    qlr_.push_back(lr); // double, as the reference's update(..., double lr)
  }
  std::vector<double> forward_noisy(std::span<const double> x, double extra) override {
    detail::check_input(x, d_in_, "forward");
    flush();
    auto xf = detail::to_f(x);
    std::vector<float> y(d_out_);
    check(xb_tile_forward_noisy(h_, xf.data(), 1, y.data(), extra));
    return detail::to_d(y);
  }
  std::vector<double> forward_with_io(std::span<const double> x, const IOParams &io) {
    detail::check_input(x, d_in_, "forward");
    flush();
    auto xf = detail::to_f(x);
    std::vector<float> y(d_out_);
    const xb_io_params c = detail::to_c(io);
    check(xb_tile_forward_io(h_, xf.data(), 1, y.data(), &c));
    return detail::to_d(y);
  }
  Matrix get_weights() const override {
    flush();
    std::vector<float> w(static_cast<size_t>(d_out_) * d_in_);
    check(xb_tile_get_weights(h_, w.data()));
    Matrix m(d_out_, d_in_);
    for (size_t k = 0; k < w.size(); ++k) m.data()[k] = w[k];
    return m;
  }
  void set_weights(const Matrix &w) override {
    if (w.rows() != d_out_ || w.cols() != d_in_)
      throw Error("set_weights: shape " + std::to_string(w.rows()) + "x" +
                  std::to_string(w.cols()) + ", expected " + std::to_string(d_out_) + "x" +
                  std::to_string(d_in_));
    flush();
    std::vector<float> f(w.data(), w.data() + w.size());
    check(xb_tile_set_weights(h_, f.data()));
  }
  void end_minibatch() override {
    flush();
    check(xb_tile_end_minibatch(h_));
  }
  std::unique_ptr<TileBase> clone() const override { return std::make_unique<AnalogTile>(*this); }

  void apply_temporal_step(const TemporalParams &tp) {
    flush();
    const xb_temporal_params c = detail::to_c(tp);
    check(xb_tile_temporal_step(h_, &c));
  }
  // proj/include/xbarsim/tile.hpp:103-104 / proj/src/tile.cpp:158-169: apply
  // already-generated trains (one sample) to the devices; flip inverts every
  // pulse.  Lines with sign 0 fire nothing (pulsed.cpp:96-112).  The GPU packs
  // a line's slots into one word, so bl <= 31.
  void apply_pulse_trains(const PulseTrains &trains, std::span<const int> sign_x,
                          std::span<const int> sign_d, bool flip_direction) {
    if (trains.x_lines != d_in_ || trains.d_lines != d_out_ ||
        static_cast<int>(sign_x.size()) != d_in_ || static_cast<int>(sign_d.size()) != d_out_)
      throw Error("apply_coincidences: trains do not conform to tile shape");
    if (trains.bl < 0 || trains.bl > 31)
      throw Error("apply_pulse_trains: bl " + std::to_string(trains.bl) +
                  " exceeds the 31 slots of a packed B200 train word");
    flush();
    auto pack = [&](int lines, std::span<const int> sign, bool is_x) {
      std::vector<uint32_t> w(static_cast<size_t>(lines), 0u);
      for (int l = 0; l < lines; ++l) {
        if (sign[l] == 0) continue;
        uint32_t v = sign[l] < 0 ? 0x80000000u : 0u;
        for (int t = 0; t < trains.bl; ++t)
          if (is_x ? trains.x_bit(t, l) : trains.d_bit(t, l)) v |= 1u << t;
        w[static_cast<size_t>(l)] = v;
      }
      return w;
    };
    const std::vector<uint32_t> xw = pack(d_in_, sign_x, true);
    const std::vector<uint32_t> dw = pack(d_out_, sign_d, false);
    check(xb_tile_apply_trains(h_, xw.data(), dw.data(), 1, flip_direction ? 1 : 0));
  }

  const TileSettings &settings() const { return settings_; }
  // proj/include/xbarsim/tile.hpp:107: the realized devices (downloaded)
  const DeviceMatrix &device() const {
    std::vector<float> up(static_cast<size_t>(d_out_) * d_in_), dn(up.size()), mx(up.size()),
        mn(up.size());
    check(xb_tile_get_device(h_, up.data(), dn.data(), mx.data(), mn.data()));
    device_ = DeviceMatrix(settings_.device, d_out_, d_in_);
    for (int i = 0; i < d_out_; ++i)
      for (int j = 0; j < d_in_; ++j) {
        const size_t k = static_cast<size_t>(i) * d_in_ + j;
        DeviceRealization &c = device_.at(i, j);
        c.dw_min_up = up[k];
        c.dw_min_down = dn[k];
        c.w_max = mx[k];
        c.w_min = mn[k];
        c.slope = settings_.device.slope; // nominal copies (device.cpp:43-44)
        c.gamma = settings_.device.gamma;
      }
    return device_;
  }
  // proj/include/xbarsim/tile.hpp:108: the stored (clipped) weights
  const Matrix &stored_weights() const {
    weights_ = get_weights();
    return weights_;
  }
  double learning_rate() const { return xb_tile_learning_rate(h_); }
  void set_learning_rate(double lr) { check(xb_tile_set_learning_rate(h_, lr)); }

  // batched extras of the B200 path: B samples per call
  void forward_batch(const float *X, int B, float *Y) override {
    flush();
    check(xb_tile_forward(h_, X, B, Y));
  }
  void forward_noisy_batch(const float *X, int B, float *Y, double extra) override {
    flush();
    check(xb_tile_forward_noisy(h_, X, B, Y, extra));
  }
  void backward_batch(const float *D, int B, float *G) override {
    flush();
    check(xb_tile_backward(h_, D, B, G));
  }
  void update_batch(const float *X, const float *D, int B, const double *lr) override {
    flush();
    check(xb_tile_update(h_, X, D, B, lr));
  }
  // applies the queued updates now (also done implicitly, see the file comment)
  // The queue is taken out BEFORE the call: if the batched update fails (a
  // CUDA error), the batch is dropped and reported once, instead of staying
  // queued and re-raising from every later call on this tile.
  void flush() const {
    if (qlr_.empty()) return;
    std::vector<float> x, d;
    std::vector<double> lr;
    x.swap(qx_);
    d.swap(qd_);
    lr.swap(qlr_);
    check(xb_tile_update(h_, x.data(), d.data(), static_cast<int>(lr.size()), lr.data()));
  }
  size_t queued_updates() const { return qlr_.size(); }
  xb_tile *handle() const { return h_; }

private:
  TileSettings settings_;
  xb_tile *h_ = nullptr;
  int d_out_ = 0, d_in_ = 0;
  bool owned_ = true;
  mutable std::vector<float> qx_, qd_;
  mutable std::vector<double> qlr_;
  mutable DeviceMatrix device_;
  mutable Matrix weights_;
};

// proj/include/xbarsim/compound.hpp:93-131, on the GPU (updates go straight
// through: transfer events interleave with samples)
class TransferTile : public TileBase {
public:
  TransferTile(int d_out, int d_in, const TransferSettings &s, uint64_t seed)
      : d_out_(d_out), d_in_(d_in), s_(s) {
    xb_transfer_config c;
    xb_default_transfer_config(&c);
    c.fast_device = detail::to_c(s.fast_device);
    c.slow_device = detail::to_c(s.slow_device);
    c.forward_io = detail::to_c(s.forward_io);
    c.backward_io = detail::to_c(s.backward_io);
    c.update = detail::to_c(s.update);
    c.temporal = detail::to_c(s.temporal);
    c.mvm_precision = static_cast<int32_t>(s.mvm_precision);
    c.transfer_every = s.transfer_every;
    c.units_in_mbatch = s.units_in_mbatch ? 1 : 0;
    c.transfer_lr = s.transfer_lr;
    c.columns_per_event = s.columns_per_event;
    c.has_transfer_io = s.has_transfer_io ? 1 : 0;
    c.gamma = s.gamma;
    c.transfer_io = detail::to_c(s.transfer_io);
    check(xb_transfer_create(&c, d_out, d_in, seed, &h_));
  }
  ~TransferTile() override {
    if (h_) xb_transfer_destroy(h_);
  }
  // proj/include/xbarsim/compound.hpp:109-111: deep copy
  TransferTile(const TransferTile &o) : d_out_(o.d_out_), d_in_(o.d_in_), s_(o.s_) {
    check(xb_transfer_clone(o.h_, &h_));
  }
  TransferTile &operator=(const TransferTile &) = delete;

  int d_out() const override { return d_out_; }
  int d_in() const override { return d_in_; }
  std::vector<double> forward(std::span<const double> x) override {
    detail::check_input(x, d_in_, "forward");
    auto xf = detail::to_f(x);
    std::vector<float> y(d_out_);
    check(xb_transfer_forward(h_, xf.data(), 1, y.data()));
    return detail::to_d(y);
  }
  std::vector<double> backward(std::span<const double> d) override {
    detail::check_input(d, d_out_, "backward");
    auto df = detail::to_f(d);
    std::vector<float> g(d_in_);
    check(xb_transfer_backward(h_, df.data(), 1, g.data()));
    return detail::to_d(g);
  }
  void update(std::span<const double> x, std::span<const double> d, double lr) override {
    detail::check_input(x, d_in_, "update(x)");
    detail::check_input(d, d_out_, "update(d)");
    auto xf = detail::to_f(x);
    auto df = detail::to_f(d);
    check(xb_transfer_update(h_, xf.data(), df.data(), 1, &lr));
  }
  // proj/src/compound.cpp:228-238
  std::vector<double> forward_noisy(std::span<const double> x, double extra) override {
    detail::check_input(x, d_in_, "forward");
    auto xf = detail::to_f(x);
    std::vector<float> y(d_out_);
    check(xb_transfer_forward_noisy(h_, xf.data(), 1, y.data(), extra));
    return detail::to_d(y);
  }
  Matrix get_weights() const override {
    std::vector<float> w(static_cast<size_t>(d_out_) * d_in_);
    check(xb_transfer_get_weights(h_, w.data()));
    Matrix m(d_out_, d_in_);
    for (size_t k = 0; k < w.size(); ++k) m.data()[k] = w[k];
    return m;
  }
  void set_weights(const Matrix &w) override {
    std::vector<float> f(w.data(), w.data() + w.size());
    check(xb_transfer_set_weights(h_, f.data()));
  }
  void end_minibatch() override { check(xb_transfer_end_minibatch(h_)); }
  std::unique_ptr<TileBase> clone() const override {
    return std::make_unique<TransferTile>(*this);
  }
  void forward_batch(const float *X, int B, float *Y) override {
    check(xb_transfer_forward(h_, X, B, Y));
  }
  void forward_noisy_batch(const float *X, int B, float *Y, double extra) override {
    check(xb_transfer_forward_noisy(h_, X, B, Y, extra));
  }
  void backward_batch(const float *D, int B, float *G) override {
    check(xb_transfer_backward(h_, D, B, G));
  }
  void update_batch(const float *X, const float *D, int B, const double *lr) override {
    check(xb_transfer_update(h_, X, D, B, lr));
  }
  void transfer_step() { check(xb_transfer_step(h_)); }
  long transfer_events() const { return xb_transfer_events(h_); }

private:
  int d_out_, d_in_;
  TransferSettings s_;
  xb_transfer *h_ = nullptr;
};

// proj/include/xbarsim/compound.hpp:15-28
enum class UnitCellPolicy { round_robin = XB_UC_ROUND_ROBIN, all_together = XB_UC_ALL_TOGETHER };
struct UnitCellSettings {
  std::vector<DeviceParams> devices;
  std::vector<double> gains;
  UnitCellPolicy policy = UnitCellPolicy::all_together;
  IOParams forward_io;
  IOParams backward_io;
  UpdateParams update;
  TemporalParams temporal;
  MvmPrecision mvm_precision = MvmPrecision::tf32x3;
};

// proj/include/xbarsim/compound.hpp:30-71, on the GPU: members are B200 tiles,
// the effective weight sum_k g_k W_k lives in HBM
class UnitCellTile : public TileBase {
public:
  UnitCellTile(int d_out, int d_in, const UnitCellSettings &s, uint64_t seed)
      : d_out_(d_out), d_in_(d_in), s_(s) {
    xb_unitcell_config c;
    xb_default_unitcell_config(&c);
    if (s.devices.empty()) throw Error("unit_cell.devices: need at least one device");
    if (s.gains.size() != s.devices.size())
      throw Error("unit_cell.gains: length must match devices");
    if (s.devices.size() > XB_MAX_CELL_DEVICES)
      throw Error("unit_cell.devices: at most " + std::to_string(XB_MAX_CELL_DEVICES) +
                  " on the B200 path");
    c.n_devices = static_cast<int32_t>(s.devices.size());
    for (size_t k = 0; k < s.devices.size(); ++k) {
      c.devices[k] = detail::to_c(s.devices[k]);
      c.gains[k] = s.gains[k];
    }
    c.policy = static_cast<int32_t>(s.policy);
    c.forward_io = detail::to_c(s.forward_io);
    c.backward_io = detail::to_c(s.backward_io);
    c.update = detail::to_c(s.update);
    c.temporal = detail::to_c(s.temporal);
    c.mvm_precision = static_cast<int32_t>(s.mvm_precision);
    check(xb_unitcell_create(&c, d_out, d_in, seed, &h_));
    bind();
  }
  UnitCellTile(const UnitCellTile &o) : d_out_(o.d_out_), d_in_(o.d_in_), s_(o.s_) {
    check(xb_unitcell_clone(o.h_, &h_));
    bind();
  }
  UnitCellTile &operator=(const UnitCellTile &) = delete;
  ~UnitCellTile() override {
    if (h_) xb_unitcell_destroy(h_);
  }

  int d_out() const override { return d_out_; }
  int d_in() const override { return d_in_; }
  // compound.cpp:82-107: length check only (no finiteness check, unlike AnalogTile)
  std::vector<double> forward(std::span<const double> x) override {
    length(x, d_in_, "forward");
    auto xf = detail::to_f(x);
    std::vector<float> y(d_out_);
    check(xb_unitcell_forward(h_, xf.data(), 1, y.data()));
    return detail::to_d(y);
  }
  std::vector<double> backward(std::span<const double> d) override {
    length(d, d_out_, "backward");
    auto df = detail::to_f(d);
    std::vector<float> g(d_in_);
    check(xb_unitcell_backward(h_, df.data(), 1, g.data()));
    return detail::to_d(g);
  }
  std::vector<double> forward_noisy(std::span<const double> x, double extra) override {
    length(x, d_in_, "forward");
    auto xf = detail::to_f(x);
    std::vector<float> y(d_out_);
    check(xb_unitcell_forward_noisy(h_, xf.data(), 1, y.data(), extra));
    return detail::to_d(y);
  }
  // compound.cpp:109-147
  void update(std::span<const double> x, std::span<const double> d, double lr) override {
    if (static_cast<int>(x.size()) != d_in_ || static_cast<int>(d.size()) != d_out_)
      throw Error("update: x/d lengths do not match tile shape");
    auto xf = detail::to_f(x);
    auto df = detail::to_f(d);
    check(xb_unitcell_update(h_, xf.data(), df.data(), 1, &lr));
  }
  Matrix get_weights() const override {
    std::vector<float> w(static_cast<size_t>(d_out_) * d_in_);
    check(xb_unitcell_get_weights(h_, w.data()));
    Matrix m(d_out_, d_in_);
    for (size_t k = 0; k < w.size(); ++k) m.data()[k] = w[k];
    return m;
  }
  void set_weights(const Matrix &w) override {
    std::vector<float> f(w.data(), w.data() + w.size());
    check(xb_unitcell_set_weights(h_, f.data()));
  }
  void end_minibatch() override { check(xb_unitcell_end_minibatch(h_)); }
  std::unique_ptr<TileBase> clone() const override {
    return std::make_unique<UnitCellTile>(*this);
  }
  void forward_batch(const float *X, int B, float *Y) override {
    check(xb_unitcell_forward(h_, X, B, Y));
  }
  void forward_noisy_batch(const float *X, int B, float *Y, double extra) override {
    check(xb_unitcell_forward_noisy(h_, X, B, Y, extra));
  }
  void backward_batch(const float *D, int B, float *G) override {
    check(xb_unitcell_backward(h_, D, B, G));
  }
  void update_batch(const float *X, const float *D, int B, const double *lr) override {
    check(xb_unitcell_update(h_, X, D, B, lr));
  }
  int n_members() const { return static_cast<int>(members_.size()); }
  // compound.hpp:53: read-only view of member k (weights, device realization)
  const AnalogTile &member(int k) const { return *members_.at(static_cast<size_t>(k)); }

private:
  static void length(std::span<const double> v, int expected, const char *what) {
    if (static_cast<int>(v.size()) != expected)
      throw Error(std::string(what) + ": length " + std::to_string(v.size()) + ", expected " +
                  std::to_string(expected));
  }
  void bind() {
    members_.clear();
    for (int k = 0; k < xb_unitcell_n_members(h_); ++k) {
      TileSettings m; // compound.cpp:31-42
      m.device = s_.devices[static_cast<size_t>(k)];
      m.forward_io = s_.forward_io;
      m.backward_io = s_.backward_io;
      m.update = s_.update;
      m.temporal = s_.temporal;
      m.mvm_precision = s_.mvm_precision;
      members_.push_back(
          std::make_unique<AnalogTile>(xb_unitcell_member(h_, k), d_out_, d_in_, m));
    }
  }
  int d_out_, d_in_;
  UnitCellSettings s_;
  xb_unitcell *h_ = nullptr;
  std::vector<std::unique_ptr<AnalogTile>> members_;
};

// ---- PCM inference, proj/include/xbarsim/inference.hpp:49-70 ----
struct ProgrammedState {
  double t0 = 0.0;
  double t = 0.0;
};

inline ProgrammedState program(AnalogTile &tile, const Matrix &w_target,
                               const InferenceNoiseModel &model, uint64_t seed) {
  if (w_target.rows() != tile.d_out() || w_target.cols() != tile.d_in())
    throw Error("program: target shape does not match tile");
  tile.flush();
  std::vector<float> f(w_target.data(), w_target.data() + w_target.size());
  const xb_inference_model m = detail::to_c(model);
  check(xb_tile_program(tile.handle(), f.data(), &m, seed));
  return ProgrammedState{model.t0, model.t0};
}

inline void drift_to(AnalogTile &tile, ProgrammedState &state, double t) {
  check(xb_tile_drift_to(tile.handle(), t));
  state.t = t;
}

inline std::vector<double> forward_with_read_noise(AnalogTile &tile, std::span<const double> x,
                                                   const InferenceNoiseModel &model) {
  return tile.forward_noisy(x, model.read_noise_scale);
}

struct DriftCompensation {
  double baseline_readout = 0.0;
};

inline DriftCompensation calibrate_compensation(AnalogTile &tile,
                                                const InferenceNoiseModel &model) {
  tile.flush();
  const xb_inference_model m = detail::to_c(model);
  double out = 0.0;
  check(xb_tile_probe_readout(tile.handle(), &m, &out));
  return DriftCompensation{out};
}

// ------------------------------------------------------------ row sharding
// Multi-GPU extension (no reference symbol: the reference tile is one device;
// SURVEY.md 8e).  A Comm joins the ranks of one logical tile: NCCL over
// NVLink/NVSwitch (unique id from rank 0, sent out of band), or an in-process
// loopback group whose members are driven by one host thread each.
class Comm {
public:
  using Id = std::array<uint8_t, XB_COMM_ID_BYTES>;
  static Id unique_id() {
    Id id{};
    check(xb_comm_unique_id(id.data()));
    return id;
  }
  // ncclCommInitRank on the current CUDA device (collective over the ranks)
  Comm(const Id &id, int nranks, int rank) { check(xb_comm_create(id.data(), nranks, rank, &h_)); }
  static std::vector<Comm> local(int nranks) {
    std::vector<xb_comm *> hs(static_cast<size_t>(nranks), nullptr);
    check(xb_comm_create_local(nranks, hs.data()));
    std::vector<Comm> out;
    for (xb_comm *h : hs) out.emplace_back(Comm(h));
    return out;
  }
  Comm(Comm &&o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  Comm &operator=(Comm &&o) noexcept {
    std::swap(h_, o.h_);
    return *this;
  }
  Comm(const Comm &) = delete;
  ~Comm() {
    if (h_) xb_comm_destroy(h_);
  }
  int size() const { return xb_comm_size(h_); }
  int rank() const { return xb_comm_rank(h_); }
  xb_comm *handle() const { return h_; }

private:
  explicit Comm(xb_comm *h) : h_(h) {}
  xb_comm *h_ = nullptr;
};

// contiguous, balanced row ranges; the first d_out % P ranks get one more row
inline std::pair<int, int> partition_rows(int d_out, int world, int rank) {
  if (world < 1 || rank < 0 || rank >= world || d_out < world)
    throw Error("partition_rows: need 0 <= rank < world <= d_out");
  const int base = d_out / world, extra = d_out % world;
  const int r0 = rank * base + std::min(rank, extra);
  return {r0, r0 + base + (rank < extra ? 1 : 0)};
}

// This rank's shard of one logical d_out x d_in AnalogTile.  x is replicated;
// d and y are this rank's rows; the backward returns the full g on every
// rank.  update and forward are bit for bit those of the unsharded tile
// (global-index random draws; max|d| and the bound-management flags are
// all-reduced); the backward differs only by the fp32 order of the
// cross-rank sum.  Host buffers, synchronous, like AnalogTile's batch calls.
class RowShardedTile {
public:
  RowShardedTile(int d_out, int d_in, const TileSettings &settings, uint64_t seed, Comm &comm)
      : d_out_(d_out), d_in_(d_in) {
    std::tie(r0_, r1_) = partition_rows(d_out, comm.size(), comm.rank());
    const xb_tile_config c = detail::to_c(settings);
    const xb_shard sh{r0_, r1_, d_out, 0};
    check(xb_tile_create(&c, d_out, d_in, seed, &sh, &h_));
    if (xb_tile_attach_comm(h_, comm.handle())) {
      const std::string msg = xb_last_error();
      xb_tile_destroy(h_);
      throw Error(msg);
    }
  }
  ~RowShardedTile() {
    if (h_) xb_tile_destroy(h_);
  }
  RowShardedTile(const RowShardedTile &) = delete;
  RowShardedTile &operator=(const RowShardedTile &) = delete;

  int d_out() const { return d_out_; }
  int d_in() const { return d_in_; }
  int row_begin() const { return r0_; }
  int row_end() const { return r1_; }
  int local_rows() const { return r1_ - r0_; }

  // W rows [row_begin, row_end), row-major
  void set_weights(const float *w_local) { check(xb_tile_set_weights(h_, w_local)); }
  std::vector<float> get_weights() const {
    std::vector<float> w(static_cast<size_t>(local_rows()) * d_in_);
    check(xb_tile_get_weights(h_, w.data()));
    return w;
  }
  // X [B][d_in] -> Y [B][local_rows]
  void forward_batch(const float *X, int B, float *Y) { check(xb_tile_forward(h_, X, B, Y)); }
  // D [B][local_rows] -> G [B][d_in] (all rows)
  void backward_batch(const float *D, int B, float *G) { check(xb_tile_backward(h_, D, B, G)); }
  // B sequential updates of the whole tile (lr[B] may be null)
  void update_batch(const float *X, const float *D, int B, const double *lr) {
    check(xb_tile_update(h_, X, D, B, lr));
  }
  xb_tile *handle() const { return h_; }

private:
  xb_tile *h_ = nullptr;
  int d_out_ = 0, d_in_ = 0, r0_ = 0, r1_ = 0;
};

inline double drift_compensation_factor(AnalogTile &tile, const DriftCompensation &comp,
                                        const InferenceNoiseModel &model) {
  tile.flush();
  const xb_inference_model m = detail::to_c(model);
  double a = 0.0;
  check(xb_tile_drift_compensation_factor(tile.handle(), comp.baseline_readout, &m, &a));
  return a;
}

} // namespace xbarsim_b200
