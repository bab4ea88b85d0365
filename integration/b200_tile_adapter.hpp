// integration/b200_tile_adapter.hpp -- the reference-side binding of the B200
// tile, compiled against the reference's own
// headers: xbarsim::B200AnalogTile implements the reference's abstract
// xbarsim::TileBase (proj/include/xbarsim/tile.hpp:47-70) over the C++ mirror
// include/xbarsim_b200/tile.hpp, which calls libxbtile.so through the C ABI.
//
// A maintainer adds this header to the reference tree and returns
// std::make_unique<B200AnalogTile>(...) from build_tile
// (proj/src/config.cpp:640-681) for a "b200" backend.  tests/test_gpu_cpp.py
// runs the reference's own NN tests (proj/tests/test_nn.cpp) with every
// AnalogTile of those tests replaced by this adapter
// (integration/test_nn_reference_on_b200.cpp).
#pragma once

#include <algorithm>
#include <memory>
#include <span>
#include <vector>

#include "xbarsim/tile.hpp"       // the reference (-I<reference>/proj/include)
#include "xbarsim_b200/tile.hpp"  // the B200 mirror (-I<repo>/include)

namespace xbarsim {

inline xbarsim_b200::IOParams to_b200(const IOParams &i) {
  xbarsim_b200::IOParams r;
  r.dac_bits = i.dac_bits;
  r.adc_bits = i.adc_bits;
  r.input_bound = i.input_bound;
  r.output_bound = i.output_bound;
  r.sigma_inp = i.sigma_inp;
  r.sigma_out = i.sigma_out;
  r.sigma_w = i.sigma_w;
  r.noise_management = static_cast<xbarsim_b200::NoiseManagement>(i.noise_management);
  r.is_perfect = i.is_perfect;
  return r;
}

inline xbarsim_b200::TileSettings to_b200(const TileSettings &s) {
  xbarsim_b200::TileSettings o;
  o.device.kind = static_cast<xbarsim_b200::DeviceKind>(s.device.kind);
  o.device.dw_min = s.device.dw_min;
  o.device.dw_min_dtod = s.device.dw_min_dtod;
  o.device.dw_min_std = s.device.dw_min_std;
  o.device.up_down = s.device.up_down;
  o.device.up_down_dtod = s.device.up_down_dtod;
  o.device.w_max = s.device.w_max;
  o.device.w_min = s.device.w_min;
  o.device.w_max_dtod = s.device.w_max_dtod;
  o.device.w_min_dtod = s.device.w_min_dtod;
  o.device.slope = s.device.slope;
  o.device.gamma = s.device.gamma;
  o.forward_io = to_b200(s.forward_io);
  o.backward_io = to_b200(s.backward_io);
  o.update.bl = s.update.bl;
  o.update.bl_management = s.update.bl_management;
  o.update.pulse_type = static_cast<xbarsim_b200::PulseType>(s.update.pulse_type);
  o.temporal.decay_rate = s.temporal.decay_rate;
  o.temporal.decay_dtod = s.temporal.decay_dtod;
  o.temporal.diffusion_sigma = s.temporal.diffusion_sigma;
  o.temporal.diffusion_dtod = s.temporal.diffusion_dtod;
  o.temporal.reset_prob = s.temporal.reset_prob;
  o.temporal.reset_dtod = s.temporal.reset_dtod;
  // the reference computes in fp64: the per-sample calls of the reference
  // API take the exact fp32 path (tcgen05 serves batches of >= 16 samples)
  o.mvm_precision = xbarsim_b200::MvmPrecision::fp32;
  return o;
}

class B200AnalogTile : public TileBase {
public:
  B200AnalogTile(int d_out, int d_in, const TileSettings &s, uint64_t seed)
      : settings_(s), t_(d_out, d_in, to_b200(s), seed) {}
  B200AnalogTile(const B200AnalogTile &o) : settings_(o.settings_), t_(o.t_) {}

  int d_out() const override { return t_.d_out(); }
  int d_in() const override { return t_.d_in(); }
  std::vector<double> forward(std::span<const double> x) override { return t_.forward(x); }
  std::vector<double> backward(std::span<const double> d) override { return t_.backward(d); }
  // queued; applied as one batched GPU update at the next read
  void update(std::span<const double> x, std::span<const double> d, double lr) override {
    t_.update(x, d, lr);
  }
  std::vector<double> forward_noisy(std::span<const double> x, double e) override {
    return t_.forward_noisy(x, e);
  }
  Matrix get_weights() const override {
    const auto w = t_.get_weights();
    Matrix m(w.rows(), w.cols());
    std::copy(w.data(), w.data() + w.size(), m.data());
    return m;
  }
  void set_weights(const Matrix &w) override {
    xbarsim_b200::Matrix m(w.rows(), w.cols());
    std::copy(w.data(), w.data() + w.size(), m.data());
    t_.set_weights(m);
  }
  void end_minibatch() override { t_.end_minibatch(); }
  std::unique_ptr<TileBase> clone() const override {
    return std::make_unique<B200AnalogTile>(*this);
  }

  // AnalogTile extras the reference's callers use (tile.hpp:95-111)
  std::vector<double> forward_with_io(std::span<const double> x, const IOParams &io) {
    return t_.forward_with_io(x, to_b200(io));
  }
  const TileSettings &settings() const { return settings_; }
  double learning_rate() const { return t_.learning_rate(); }
  void set_learning_rate(double lr) { t_.set_learning_rate(lr); }
  xbarsim_b200::AnalogTile &b200() { return t_; }

private:
  TileSettings settings_;
  xbarsim_b200::AnalogTile t_;
};

} // namespace xbarsim
