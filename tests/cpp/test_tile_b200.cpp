// C++ parity driver for the B200 host layer (include/xbarsim_b200/tile.hpp):
// the reference's own unit tests (proj/tests/test_pulsed.cpp, test_tile.cpp,
// test_compounds.cpp, test_inference.cpp) re-run through the C++ API on the
// GPU.  Prints one line per case and exits non-zero on any failure; run by
// tests/test_gpu_cpp.py.
#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "xbarsim_b200/tile.hpp"

using namespace xbarsim_b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                                        \
  do {                                                                                     \
    ++g_checks;                                                                            \
    if (!(cond)) {                                                                         \
      ++g_fail;                                                                            \
      std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);                \
    }                                                                                      \
  } while (0)

template <class F> static bool throws(F f, const char *needle = nullptr) {
  try {
    f();
  } catch (const Error &e) {
    return needle == nullptr || std::string(e.what()).find(needle) != std::string::npos;
  }
  return false;
}

static IOParams io_off() { // proj/tests/helpers.hpp:56-68
  IOParams io;
  io.dac_bits = 0;
  io.adc_bits = 0;
  io.input_bound = 1e9;
  io.output_bound = 1e9;
  io.sigma_out = 0.0;
  io.noise_management = NoiseManagement::none;
  return io;
}

static TileSettings quiet_settings(double dw_min = 0.001, double bound = 1.0) {
  TileSettings s;
  s.device.dw_min = dw_min;
  s.device.w_max = bound;
  s.device.w_min = -bound;
  s.forward_io = io_off();
  s.backward_io = io_off();
  return s;
}

static Matrix random_matrix(int r, int c, double scale, uint64_t seed) {
  std::mt19937_64 g(seed);
  std::uniform_real_distribution<double> u(-scale, scale);
  Matrix m(r, c);
  for (size_t k = 0; k < m.size(); ++k) m.data()[k] = u(g);
  return m;
}

static void run(const char *name, const std::function<void()> &f) {
  const int before = g_fail;
  try {
    f();
  } catch (const std::exception &e) {
    ++g_fail;
    std::printf("  exception: %s\n", e.what());
  }
  std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", name);
}

int main() {
  run("saturated trains give -31 dw_min (test_pulsed.cpp:66-79)", [] {
    AnalogTile tile(1, 1, quiet_settings(0.001, 1.0), 2);
    tile.update(std::vector<double>{1.0}, std::vector<double>{-1.0}, 10.0);
    CHECK(tile.queued_updates() == 1);
    CHECK(std::fabs(tile.get_weights()(0, 0) + 0.031) < 1e-7);
    CHECK(tile.queued_updates() == 0);
  });
  run("no-op updates (test_pulsed.cpp:177-189)", [] {
    AnalogTile tile(2, 2, quiet_settings(), 11);
    tile.set_weights(random_matrix(2, 2, 0.3, 12));
    Matrix before = tile.get_weights();
    tile.update(std::vector<double>{1, 1}, std::vector<double>{1, 1}, 0.0);
    tile.update(std::vector<double>{0, 0}, std::vector<double>{1, 1}, 0.1);
    tile.update(std::vector<double>{1, 1}, std::vector<double>{0, 0}, 0.1);
    CHECK(tile.get_weights() == before);
  });
  run("perfect forward is the exact mat-vec (test_tile.cpp:53-64)", [] {
    TileSettings s = quiet_settings();
    s.forward_io = perfect_io();
    AnalogTile tile(2, 2, s, 42);
    Matrix w(2, 2);
    w(0, 0) = 1.0;
    w(1, 1) = 1.0;
    tile.set_weights(w);
    auto y = tile.forward(std::vector<double>{0.3, -0.2});
    CHECK(std::fabs(y[0] - 0.3) < 1e-7 && std::fabs(y[1] + 0.2) < 1e-7);
  });
  run("set/get clip (test_tile.cpp:268-291)", [] {
    TileSettings s = quiet_settings(0.001, 1.0);
    s.forward_io.sigma_out = 0.1;
    s.forward_io.sigma_w = 0.1;
    AnalogTile tile(2, 2, s, 11);
    Matrix w(2, 2);
    w(0, 0) = 0.5;
    w(0, 1) = -0.25;
    w(1, 0) = 10.0;
    tile.set_weights(w);
    Matrix got = tile.get_weights();
    CHECK(got(0, 0) == 0.5 && got(0, 1) == -0.25 && got(1, 0) == 1.0 && got(1, 1) == 0.0);
    for (int t = 0; t < 50; ++t) tile.forward(std::vector<double>{0.3, 0.4});
    CHECK(tile.get_weights() == got);
  });
  run("errors name the field (test_tile.cpp:293-305)", [] {
    AnalogTile tile(2, 3, quiet_settings(), 12);
    CHECK(throws([&] { tile.forward(std::vector<double>{1.0, 2.0}); }, "forward: length 2"));
    CHECK(throws([&] { tile.backward(std::vector<double>{1.0, 2.0, 3.0}); }, "backward"));
    CHECK(throws([&] { tile.forward(std::vector<double>{1.0, NAN, 0.0}); }, "non-finite"));
    CHECK(throws([&] { tile.set_weights(Matrix(3, 2, 0.0)); }, "set_weights: shape"));
    CHECK(throws([&] { tile.set_learning_rate(0.0); }, "learning_rate"));
    CHECK(throws([&] {
      tile.update(std::vector<double>{1, 1, 1}, std::vector<double>{1, 1}, -0.5);
    }, "learning rate must be > 0"));
    TileSettings bad = quiet_settings();
    bad.device.dw_min = -1.0;
    CHECK(throws([&] { AnalogTile t(2, 2, bad, 1); }, "device.dw_min"));
  });
  run("mean update equals lr d x^T through the queue (test_pulsed.cpp:203-231)", [] {
    AnalogTile tile(4, 4, quiet_settings(0.001, 1000.0), 14);
    const std::vector<double> x = {1.0, -0.8, 0.6, 0.4}, d = {0.9, -0.7, 0.5, 0.3};
    const int n = 4000;
    for (int t = 0; t < n; ++t) tile.update(x, d, 0.01); // one batched kernel call
    Matrix w = tile.get_weights();
    double worst = 0.0;
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j)
        if (std::fabs(d[i] * x[j]) > 0.1)
          worst = std::max(worst, std::fabs(w(i, j) / n - 0.01 * d[i] * x[j]) /
                                      std::fabs(0.01 * d[i] * x[j]));
    CHECK(worst < 0.04);
  });
  run("deferred queue == immediate batched update (deterministic pulses)", [] {
    TileSettings s = quiet_settings(0.001, 10.0);
    s.update.pulse_type = PulseType::deterministic_implicit;
    AnalogTile a(3, 5, s, 3);
    AnalogTile b(3, 5, s, 3);
    std::vector<float> X, D;
    std::vector<double> L;
    for (int t = 0; t < 7; ++t) {
      auto x = random_matrix(1, 5, 1.0, 100 + t), d = random_matrix(1, 3, 1.0, 200 + t);
      std::vector<double> xs(x.data(), x.data() + 5), ds(d.data(), d.data() + 3);
      a.update(xs, ds, 0.02);
      X.insert(X.end(), xs.begin(), xs.end());
      D.insert(D.end(), ds.begin(), ds.end());
      L.push_back(0.02);
    }
    b.update_batch(X.data(), D.data(), 7, L.data());
    CHECK(a.get_weights() == b.get_weights());
  });
  run("clone is a deep copy (tile.hpp:91)", [] {
    AnalogTile a(3, 3, quiet_settings(), 5);
    a.set_weights(random_matrix(3, 3, 0.3, 6));
    auto c = a.clone();
    a.update(std::vector<double>{1, 1, 1}, std::vector<double>{1, 1, 1}, 1.0);
    CHECK(!(c->get_weights() == a.get_weights()));
  });
  run("transfer schedule fires floor(N / transfer_every) events (test_compounds.cpp)", [] {
    TransferSettings s;
    s.forward_io = io_off();
    s.backward_io = io_off();
    s.transfer_every = 3;
    TransferTile t(2, 2, s, 15);
    for (int k = 0; k < 10; ++k)
      t.update(std::vector<double>{1.0, 0.5}, std::vector<double>{0.8, -0.6}, 0.05);
    CHECK(t.transfer_events() == 3);
    TransferSettings m = s;
    m.transfer_every = 1;
    m.units_in_mbatch = true;
    TransferTile u(2, 2, m, 16);
    for (int k = 0; k < 4; ++k)
      u.update(std::vector<double>{1.0, 0.5}, std::vector<double>{0.8, -0.6}, 0.05);
    CHECK(u.transfer_events() == 0);
    u.end_minibatch();
    CHECK(u.transfer_events() == 1);
  });
  run("zero programming noise writes the target; uniform drift (test_inference.cpp)", [] {
    TileSettings s = quiet_settings(0.001, 100.0);
    s.forward_io = perfect_io();
    AnalogTile tile(2, 2, s, 11);
    InferenceNoiseModel m;
    m.prog_noise_scale = 0.0;
    m.nu_std = 0.0;
    m.nu_mean = 0.06;
    m.t0 = 1.0;
    Matrix target = random_matrix(2, 2, 0.5, 12);
    ProgrammedState st = program(tile, target, m, 13);
    Matrix w = tile.get_weights();
    for (int k = 0; k < 4; ++k) CHECK(std::fabs(w.data()[k] - target.data()[k]) < 1e-7);
    drift_to(tile, st, 100.0);
    w = tile.get_weights();
    const double f = std::pow(100.0, -0.06);
    for (int k = 0; k < 4; ++k) CHECK(std::fabs(w.data()[k] - target.data()[k] * f) < 1e-6);
    CHECK(throws([&] { drift_to(tile, st, 0.5); }, "drift_to: t < t0"));
  });
  run("apply_pulse_trains: saturated, flipped and zero-sign lines (test_pulsed.cpp:66-79)", [] {
    AnalogTile t(3, 2, quiet_settings(0.001, 1.0), 21);
    PulseTrains tr;
    tr.bl = 31;
    tr.x_lines = 2;
    tr.d_lines = 3;
    tr.x_bits.assign(31 * 2, 1);
    tr.d_bits.assign(31 * 3, 1);
    const std::vector<int> sx{1, 1}, sd{-1, 1, 0};
    t.apply_pulse_trains(tr, sx, sd, false);
    Matrix w = t.stored_weights();
    for (int j = 0; j < 2; ++j) {
      CHECK(std::fabs(w(0, j) + 31 * 0.001) < 1e-6);
      CHECK(std::fabs(w(1, j) - 31 * 0.001) < 1e-6);
      CHECK(w(2, j) == 0.0);
    }
    t.apply_pulse_trains(tr, sx, sd, true); // flip undoes it (constant step)
    w = t.get_weights();
    for (int k = 0; k < 6; ++k) CHECK(std::fabs(w.data()[k]) < 1e-6);
    tr.bl = 40;
    CHECK(throws([&] { t.apply_pulse_trains(tr, sx, sd, false); }, "31 slots"));
  });
  run("device(): nominal realization 1.1 / 0.9 dw_min (test_devices.cpp:17-31)", [] {
    TileSettings s = quiet_settings(0.002, 0.6);
    s.device.up_down = 0.1;
    AnalogTile t(4, 3, s, 22);
    const DeviceMatrix &dm = t.device();
    CHECK(dm.rows() == 4 && dm.cols() == 3);
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 3; ++j) {
        CHECK(std::fabs(dm.at(i, j).dw_min_up - 0.0022) < 1e-9);
        CHECK(std::fabs(dm.at(i, j).dw_min_down - 0.0018) < 1e-9);
        CHECK(std::fabs(dm.at(i, j).w_max - 0.6) < 1e-7);
        CHECK(std::fabs(dm.at(i, j).w_min + 0.6) < 1e-7);
      }
    CHECK(dm.clip(0, 0, 5.0) == dm.at(0, 0).w_max);
  });
  run("TransferTile clone and forward_noisy (compound.hpp:109-111, compound.cpp:228-238)", [] {
    TransferSettings s;
    s.forward_io = io_off();
    s.backward_io = io_off();
    s.fast_device = device_preset("reram_sb");
    s.slow_device = device_preset("reram_sb");
    s.transfer_every = 2;
    s.gamma = 0.5;
    TransferTile a(4, 3, s, 31);
    a.set_weights(random_matrix(4, 3, 0.2, 32));
    for (int k = 0; k < 3; ++k)
      a.update(std::vector<double>{1.0, -0.5, 0.25}, std::vector<double>{0.8, -0.6, 0.1, 0.3},
               0.05);
    auto c = a.clone();
    for (int k = 0; k < 5; ++k) {
      const std::vector<double> x{0.3, 0.7, -0.2}, d{-0.4, 0.9, 0.2, -0.1};
      a.update(x, d, 0.05);
      c->update(x, d, 0.05);
    }
    CHECK(a.get_weights() == c->get_weights());
    const std::vector<double> x{0.5, -0.25, 1.0};
    CHECK(a.forward_noisy(x, 0.0) == a.forward(x));
    CHECK(!(a.forward_noisy(x, 0.1) == a.forward(x)));
  });
  run("UnitCellTile: set/get, mirror pair, round robin, clone (test_compounds.cpp:43-150)", [] {
    DeviceParams d;
    d.dw_min = 1.0 / 1024;
    d.w_max = 8.0;
    d.w_min = -8.0;
    UnitCellSettings s;
    s.devices = {d, d};
    s.gains = {1.0, -1.0};
    s.forward_io = io_off();
    s.backward_io = io_off();
    UnitCellTile u(3, 4, s, 41);
    CHECK(u.n_members() == 2);
    Matrix w = random_matrix(3, 4, 0.5, 42);
    u.set_weights(w);
    Matrix e = u.get_weights();
    for (size_t k = 0; k < w.size(); ++k) CHECK(std::fabs(e.data()[k] - w.data()[k]) < 1e-6);
    const Matrix base = u.member(0).get_weights(); // fp32-stored w
    for (int k = 0; k < 5; ++k)
      u.update(std::vector<double>{1.0, -0.5, 0.25, 0.8}, std::vector<double>{0.7, -0.3, 0.9},
               0.05);
    Matrix m0 = u.member(0).get_weights(), m1 = u.member(1).get_weights();
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 4; ++j) CHECK(std::fabs(m1(i, j) + (m0(i, j) - base(i, j))) < 1e-6);
    auto c = u.clone();
    CHECK(c->get_weights() == u.get_weights());
    s.gains = {0.0, 1.0};
    UnitCellTile z(2, 2, s, 43);
    CHECK(throws([&] { z.set_weights(Matrix(2, 2, 1.0)); }, "zero first gain"));
    CHECK(throws([&] { u.update(std::vector<double>{1.0}, std::vector<double>{1.0}, 0.1); },
                 "x/d lengths"));
  });
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
