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

#include "xbarsim/compound.hpp"   // the reference (-I<reference>/proj/include)
#include "xbarsim/tile.hpp"
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

inline xbarsim_b200::DeviceParams to_b200(const DeviceParams &d) {
  xbarsim_b200::DeviceParams o;
  o.kind = static_cast<xbarsim_b200::DeviceKind>(d.kind);
  o.dw_min = d.dw_min;
  o.dw_min_dtod = d.dw_min_dtod;
  o.dw_min_std = d.dw_min_std;
  o.up_down = d.up_down;
  o.up_down_dtod = d.up_down_dtod;
  o.w_max = d.w_max;
  o.w_min = d.w_min;
  o.w_max_dtod = d.w_max_dtod;
  o.w_min_dtod = d.w_min_dtod;
  o.slope = d.slope;
  o.gamma = d.gamma;
  return o;
}

inline xbarsim_b200::UpdateParams to_b200(const UpdateParams &u) {
  xbarsim_b200::UpdateParams o;
  o.bl = u.bl;
  o.bl_management = u.bl_management;
  o.pulse_type = static_cast<xbarsim_b200::PulseType>(u.pulse_type);
  return o;
}

inline xbarsim_b200::TemporalParams to_b200(const TemporalParams &t) {
  xbarsim_b200::TemporalParams o;
  o.decay_rate = t.decay_rate;
  o.decay_dtod = t.decay_dtod;
  o.diffusion_sigma = t.diffusion_sigma;
  o.diffusion_dtod = t.diffusion_dtod;
  o.reset_prob = t.reset_prob;
  o.reset_dtod = t.reset_dtod;
  return o;
}

// the reference computes in fp64: the per-sample calls of the reference API
// take the exact fp32 path (tcgen05 serves batches of >= 16 samples)
inline xbarsim_b200::TileSettings to_b200(const TileSettings &s) {
  xbarsim_b200::TileSettings o;
  o.device = to_b200(s.device);
  o.forward_io = to_b200(s.forward_io);
  o.backward_io = to_b200(s.backward_io);
  o.update = to_b200(s.update);
  o.temporal = to_b200(s.temporal);
  o.mvm_precision = xbarsim_b200::MvmPrecision::fp32;
  return o;
}

// proj/include/xbarsim/compound.hpp:76-91
inline xbarsim_b200::TransferSettings to_b200(const TransferSettings &s) {
  xbarsim_b200::TransferSettings o;
  o.fast_device = to_b200(s.fast_device);
  o.slow_device = to_b200(s.slow_device);
  o.forward_io = to_b200(s.forward_io);
  o.backward_io = to_b200(s.backward_io);
  o.update = to_b200(s.update);
  o.temporal = to_b200(s.temporal);
  o.transfer_every = s.transfer_every;
  o.units_in_mbatch = s.units_in_mbatch;
  o.transfer_lr = s.transfer_lr;
  o.columns_per_event = s.columns_per_event;
  o.gamma = s.gamma;
  o.has_transfer_io = s.transfer_io.has_value();
  if (s.transfer_io) o.transfer_io = to_b200(*s.transfer_io);
  o.mvm_precision = xbarsim_b200::MvmPrecision::fp32;
  return o;
}

// proj/include/xbarsim/compound.hpp:19-29
inline xbarsim_b200::UnitCellSettings to_b200(const UnitCellSettings &s) {
  xbarsim_b200::UnitCellSettings o;
  for (const DeviceParams &d : s.devices) o.devices.push_back(to_b200(d));
  o.gains = s.gains;
  o.policy = s.policy == UnitCellPolicy::round_robin ? xbarsim_b200::UnitCellPolicy::round_robin
                                                     : xbarsim_b200::UnitCellPolicy::all_together;
  o.forward_io = to_b200(s.forward_io);
  o.backward_io = to_b200(s.backward_io);
  o.update = to_b200(s.update);
  o.temporal = to_b200(s.temporal);
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

// a compound tile of the mirror (TransferTile, UnitCellTile) behind the
// reference's TileBase: the same forwarding as B200AnalogTile
template <class Mirror, class Settings> class B200CompoundTile : public TileBase {
public:
  B200CompoundTile(int d_out, int d_in, const Settings &s, uint64_t seed)
      : t_(d_out, d_in, to_b200(s), seed) {}
  B200CompoundTile(const B200CompoundTile &o) : t_(o.t_) {}

  int d_out() const override { return t_.d_out(); }
  int d_in() const override { return t_.d_in(); }
  std::vector<double> forward(std::span<const double> x) override { return t_.forward(x); }
  std::vector<double> backward(std::span<const double> d) override { return t_.backward(d); }
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
    return std::make_unique<B200CompoundTile>(*this);
  }

private:
  Mirror t_;
};

using B200TransferTile = B200CompoundTile<xbarsim_b200::TransferTile, TransferSettings>;
using B200UnitCellTile = B200CompoundTile<xbarsim_b200::UnitCellTile, UnitCellSettings>;

} // namespace xbarsim
