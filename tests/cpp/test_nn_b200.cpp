// C++ driver for the batched NN host (include/xbarsim_b200/nn.hpp): the
// reference's own NN unit tests (proj/tests/test_nn.cpp) re-run on the GPU
// tiles, plus batched-vs-per-sample equivalence.  fp32 tile storage replaces
// the reference's exact double comparisons by 1e-6-scale tolerances.  Prints
// one line per case; exits non-zero on failure; run by tests/test_gpu_cpp.py.
#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "xbarsim_b200/nn.hpp"

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

// proj/tests/helpers.hpp:56-107
static IOParams io_off() {
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
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < c; ++j) m(i, j) = u(g);
  return m;
}
static std::vector<double> random_vector(int n, double scale, uint64_t seed) {
  std::mt19937_64 g(seed);
  std::uniform_real_distribution<double> u(-scale, scale);
  std::vector<double> v(static_cast<size_t>(n));
  for (double &x : v) x = u(g);
  return v;
}
static std::unique_ptr<AnalogTile> perfect_tile(int rows, int cols, uint64_t seed,
                                                double bound = 4.0) {
  TileSettings s = quiet_settings(0.001, bound);
  s.forward_io = perfect_io();
  s.backward_io = perfect_io();
  return std::make_unique<AnalogTile>(rows, cols, s, seed);
}
static std::unique_ptr<AnalogDenseLayer> make_dense(int in, int out, uint64_t seed,
                                                    Activation act = Activation::identity,
                                                    HwAwareParams hw = {}) {
  return std::make_unique<AnalogDenseLayer>(perfect_tile(out, in, seed), in, out,
                                            BiasMode::digital, act, hw);
}
static bool near(double a, double b, double tol) { return std::fabs(a - b) <= tol; }

int main() {
  run("RngStream reproduces the reference streams bit for bit (rng.cpp)", [] {
    RngStream r(123);
    CHECK(r.uniform() == 0.47542931821661116);
    CHECK(r.uniform() == 0.8734455087098733);
    RngStream g = RngStream(123).derive("blob_samples", 7);
    CHECK(g.gauss() == -2.1583929113344023);
    CHECK(g.gauss() == -0.07555836727328545);
    CHECK(g.gauss() == 0.7149513505935506);
  });
  run("a perfect dense layer is an exact affine map (test_nn.cpp:105-117)", [] {
    auto layer = make_dense(3, 2, 1);
    Matrix w = random_matrix(2, 3, 0.4, 2);
    layer->tile().set_weights(w);
    layer->set_bias(std::vector<double>{0.1, -0.2});
    std::vector<double> x = random_vector(3, 0.8, 3);
    auto y = layer->forward(x, false);
    for (int i = 0; i < 2; ++i) {
      double e = 0.0;
      for (int j = 0; j < 3; ++j) e += w(i, j) * x[static_cast<size_t>(j)];
      CHECK(near(y[static_cast<size_t>(i)], e + (i == 0 ? 0.1 : -0.2), 1e-6));
    }
  });
  run("an analog bias column is a weight on a constant input (test_nn.cpp:119-133)", [] {
    AnalogDenseLayer layer(perfect_tile(2, 4, 4), 3, 2, BiasMode::analog, Activation::identity,
                           HwAwareParams{});
    Matrix w(2, 4);
    w(0, 3) = 0.25;
    w(1, 3) = -0.5;
    layer.tile().set_weights(w);
    auto y = layer.forward(std::vector<double>{0.0, 0.0, 0.0}, false);
    CHECK(y[0] == 0.25 && y[1] == -0.5);
    CHECK(throws([] {
      AnalogDenseLayer bad(perfect_tile(2, 3, 5), 3, 2, BiasMode::analog, Activation::identity,
                           HwAwareParams{});
    }, "does not match layer"));
  });
  run("conv forward matches a naive convolution (test_nn.cpp:135-182)", [] {
    const int cin = 2, cout = 3, k = 3, h = 5, wd = 4, stride = 2, pad = 1;
    AnalogConv2DLayer conv(perfect_tile(cout, cin * k * k, 6), cin, cout, k, stride, pad, h, wd,
                           BiasMode::digital, Activation::identity, HwAwareParams{});
    Matrix w = random_matrix(cout, cin * k * k, 0.4, 7);
    conv.tile().set_weights(w);
    std::vector<double> x = random_vector(cin * h * wd, 0.9, 8);
    auto y = conv.forward(x, false);
    const int oh = conv.out_h(), ow = conv.out_w();
    CHECK(oh == 3 && ow == 2);
    for (int c = 0; c < cout; ++c)
      for (int oy = 0; oy < oh; ++oy)
        for (int ox = 0; ox < ow; ++ox) {
          double acc = 0.0;
          for (int ci = 0; ci < cin; ++ci)
            for (int ky = 0; ky < k; ++ky)
              for (int kx = 0; kx < k; ++kx) {
                const int iy = oy * stride + ky - pad, ix = ox * stride + kx - pad;
                if (iy < 0 || iy >= h || ix < 0 || ix >= wd) continue;
                acc += w(c, (ci * k + ky) * k + kx) * x[static_cast<size_t>((ci * h + iy) * wd + ix)];
              }
          CHECK(near(y[static_cast<size_t>((c * oh + oy) * ow + ox)], acc, 1e-5));
        }
  });
  run("perfect backward produces W^T grad (test_nn.cpp:204-221)", [] {
    HwAwareParams hw;
    hw.perfect_backward = true;
    auto layer = make_dense(3, 2, 12, Activation::identity, hw);
    layer->tile().set_weights(random_matrix(2, 3, 0.4, 13));
    Matrix w = layer->tile().get_weights();
    layer->forward(random_vector(3, 0.8, 14), true);
    std::vector<double> g = {0.5, -0.25};
    auto gin = layer->backward(g);
    for (int j = 0; j < 3; ++j) CHECK(gin[static_cast<size_t>(j)] == w(0, j) * 0.5 + w(1, j) * -0.25);
    CHECK(throws([&] { layer->backward(g); }, "no cached forward"));
  });
  run("input gradients match finite differences, dense and conv (test_nn.cpp:223-282)", [] {
    HwAwareParams hw;
    hw.perfect_backward = true;
    for (int conv = 0; conv < 2; ++conv) {
      Network net;
      if (conv) {
        net.add(std::make_unique<AnalogConv2DLayer>(perfect_tile(2, 9, 80), 1, 2, 3, 1, 1, 4, 4,
                                                    BiasMode::digital, Activation::tanh_act, hw));
      } else {
        net.add(make_dense(4, 5, 15, Activation::tanh_act, hw));
        net.add(make_dense(5, 3, 16, Activation::identity, hw));
      }
      initialize_network(net, 17);
      std::vector<double> x = random_vector(net.in_size(), 0.7, 18);
      std::vector<double> target = random_vector(net.out_size(), 0.5, 19);
      auto loss_at = [&](const std::vector<double> &in) {
        return loss_mse(net.forward(in, false), target).loss;
      };
      auto y = net.forward(x, true);
      auto analytic = net.backward(loss_mse(y, target).grad);
      const double eps = 1e-2; // fp32 tile outputs: a wide stencil
      for (size_t j = 0; j < x.size(); ++j) {
        std::vector<double> xp(x), xm(x);
        xp[j] += eps;
        xm[j] -= eps;
        const double fd = (loss_at(xp) - loss_at(xm)) / (2.0 * eps);
        CHECK(std::fabs(analytic[j] - fd) <= 2e-3 * std::max(1.0, std::fabs(fd)));
      }
    }
  });
  run("zero gradients leave the weights unchanged; perfect update is SGD (test_nn.cpp:315-347)",
      [] {
        auto layer = make_dense(3, 2, 23);
        layer->tile().set_weights(random_matrix(2, 3, 0.4, 24));
        Matrix before = layer->tile().get_weights();
        layer->forward(random_vector(3, 0.8, 25), true);
        layer->backward(std::vector<double>{0.0, 0.0});
        layer->apply_updates(0.1, 1);
        layer->end_minibatch();
        CHECK(layer->tile().get_weights() == before);
        HwAwareParams hw;
        hw.perfect_update = true;
        auto p = make_dense(3, 2, 26, Activation::identity, hw);
        p->tile().set_weights(random_matrix(2, 3, 0.3, 27));
        Matrix w0 = p->tile().get_weights();
        std::vector<double> x = random_vector(3, 0.8, 28);
        p->forward(x, true);
        p->backward(std::vector<double>{0.4, -0.2});
        p->apply_updates(0.05, 1);
        Matrix w = p->tile().get_weights();
        for (int i = 0; i < 2; ++i)
          for (int j = 0; j < 3; ++j)
            CHECK(near(w(i, j), w0(i, j) - 0.05 * (i == 0 ? 0.4 : -0.2) * x[static_cast<size_t>(j)],
                       1e-7));
      });
  run("weight noise is added for the batch and removed bit-exactly (test_nn.cpp:349-367)", [] {
    HwAwareParams hw;
    hw.weight_noise_sigma = 0.1;
    auto layer = make_dense(3, 2, 29, Activation::identity, hw);
    layer->tile().set_weights(random_matrix(2, 3, 0.3, 30));
    Matrix before = layer->tile().get_weights();
    RngStream noise(31);
    layer->begin_minibatch(noise);
    CHECK(!(layer->tile().get_weights() == before));
    layer->forward(random_vector(3, 0.8, 32), true);
    layer->backward(std::vector<double>{0.3, -0.1});
    layer->remove_weight_noise();
    layer->apply_updates(0.0, 1);
    layer->end_minibatch();
    CHECK(layer->tile().get_weights() == before);
  });
  run("a batched pass equals B per-sample passes on stationary weights", [] {
    Network net;
    net.add(make_dense(6, 5, 60, Activation::sigmoid));
    net.add(std::make_unique<AnalogConv2DLayer>(perfect_tile(2, 5, 61), 5, 2, 1, 1, 0, 1, 1,
                                                BiasMode::digital, Activation::tanh_act,
                                                HwAwareParams{}));
    initialize_network(net, 62);
    const int B = 9;
    std::vector<double> X(static_cast<size_t>(B) * 6);
    for (size_t k = 0; k < X.size(); ++k) X[k] = std::sin(0.37 * static_cast<double>(k));
    auto Y = net.forward_batch(X.data(), B, false);
    for (int b = 0; b < B; ++b) {
      auto y = net.forward(std::span<const double>(X.data() + b * 6, 6), false);
      for (int i = 0; i < 2; ++i) CHECK(near(y[static_cast<size_t>(i)], Y[static_cast<size_t>(b * 2 + i)], 1e-6));
    }
  });
  run("training an analog linear layer solves a separable task (test_nn.cpp:369-395)", [] {
    Network net;
    net.add(std::make_unique<AnalogDenseLayer>(
        std::make_unique<AnalogTile>(2, 4, quiet_settings(0.001, 1.0), 33), 4, 2,
        BiasMode::digital, Activation::identity, HwAwareParams{}));
    initialize_network(net, 34);
    Dataset data = make_blobs(100, 4, 2, 0.05, 35);
    TrainConfig cfg;
    cfg.loss = Loss::mse;
    cfg.lr = 0.1;
    cfg.epochs = 100;
    cfg.batch_size = 10;
    cfg.seed = 36;
    auto history = train(net, data, cfg);
    CHECK(history.back().loss < 0.01);
    CHECK(history.back().accuracy == 1.0);
    double early = 0.0, late = 0.0;
    for (int e = 0; e < 20; ++e) {
      early += history[static_cast<size_t>(e)].loss;
      late += history[static_cast<size_t>(80 + e)].loss;
    }
    CHECK(late < early);
    CHECK(evaluate_accuracy(net, make_blobs(200, 4, 2, 0.05, 35, 1)) == 1.0);
  });
  run("zero learning rate freezes the loss history (test_nn.cpp:397-417)", [] {
    TileSettings s = quiet_settings(0.001, 1.0);
    s.forward_io = perfect_io();
    s.backward_io = perfect_io();
    Network net;
    net.add(std::make_unique<AnalogDenseLayer>(std::make_unique<AnalogTile>(2, 4, s, 37), 4, 2,
                                               BiasMode::digital, Activation::identity,
                                               HwAwareParams{}));
    initialize_network(net, 38);
    TrainConfig cfg;
    cfg.lr = 0.0;
    cfg.epochs = 5;
    cfg.batch_size = 10;
    cfg.seed = 40;
    auto h = train(net, make_blobs(40, 4, 2, 0.05, 39), cfg);
    for (const EpochStats &e : h) CHECK(std::fabs(e.loss - h[0].loss) <= 1e-9 * h[0].loss);
  });
  run("reram devices stay within 5x of the digital loss; conv+dense cross-entropy MLP", [] {
    Dataset data = make_blobs(100, 4, 2, 0.05, 41);
    double digital = 0.0;
    {
      TileSettings s = quiet_settings(0.001, 1.0);
      s.forward_io = perfect_io();
      s.backward_io = perfect_io();
      HwAwareParams hw;
      hw.perfect_backward = hw.perfect_update = true;
      Network net;
      net.add(std::make_unique<AnalogDenseLayer>(std::make_unique<AnalogTile>(2, 4, s, 42), 4,
                                                 2, BiasMode::digital, Activation::identity, hw));
      initialize_network(net, 43);
      TrainConfig cfg;
      cfg.lr = 0.1;
      cfg.epochs = 60;
      cfg.seed = 44;
      digital = train(net, data, cfg).back().loss;
    }
    double analog = 0.0;
    for (int sd = 0; sd < 5; ++sd) {
      TileSettings s;
      s.device = device_preset("reram_sb");
      s.forward_io = io_off();
      s.forward_io.sigma_out = 0.02;
      s.backward_io = io_off();
      s.backward_io.sigma_out = 0.02;
      Network net;
      net.add(std::make_unique<AnalogDenseLayer>(std::make_unique<AnalogTile>(2, 4, s, 45 + sd),
                                                 4, 2, BiasMode::digital, Activation::identity,
                                                 HwAwareParams{}));
      initialize_network(net, 50 + static_cast<uint64_t>(sd));
      TrainConfig cfg;
      cfg.lr = 0.05;
      cfg.epochs = 60;
      cfg.seed = 55 + static_cast<uint64_t>(sd);
      analog += train(net, data, cfg).back().loss;
    }
    CHECK(analog / 5 < 5.0 * digital + 0.01);
    // conv -> dense -> dense with CE loss on default IO (DAC/ADC, output noise)
    // and ConstantStep devices; digital reference reaches 0.99 here
    Network mlp;
    TileSettings s;
    mlp.add(std::make_unique<AnalogConv2DLayer>(std::make_unique<AnalogTile>(4, 9, s, 70), 1, 4,
                                                3, 1, 0, 4, 4, BiasMode::digital,
                                                Activation::relu, HwAwareParams{}));
    mlp.add(std::make_unique<AnalogDenseLayer>(std::make_unique<AnalogTile>(8, 16, s, 71), 16, 8,
                                               BiasMode::digital, Activation::sigmoid,
                                               HwAwareParams{}));
    mlp.add(std::make_unique<AnalogDenseLayer>(std::make_unique<AnalogTile>(3, 8, s, 72), 8, 3,
                                               BiasMode::digital, Activation::identity,
                                               HwAwareParams{}));
    initialize_network(mlp, 73);
    TrainConfig cfg;
    cfg.loss = Loss::cross_entropy;
    cfg.lr = 0.1;
    cfg.epochs = 60;
    cfg.batch_size = 16;
    cfg.seed = 74;
    auto h = train(mlp, make_blobs(96, 16, 3, 0.2, 75), cfg);
    std::printf("  conv-dense-dense CE: loss %.4f -> %.4f, accuracy %.3f -> %.3f\n",
                h.front().loss, h.back().loss, h.front().accuracy, h.back().accuracy);
    CHECK(h.back().loss < 0.5 * h.front().loss);
    CHECK(h.back().accuracy > 0.8); // chance is 1/3
  });
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
