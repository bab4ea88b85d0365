// xbarsim_b200/nn.hpp -- the reference's NN host (proj/include/xbarsim/nn.hpp,
// proj/src/nn.cpp) over the batched B200 tile API.
//
// Same class names, constructors, switches and error messages as the
// reference.  What changes is the execution: a mini-batch goes through each
// layer as ONE batched call (forward_batch / backward_batch on the tile, one
// weight-stationary update_batch of every queued sample or conv patch),
// instead of one tile call per sample and per patch.  This is exactly the
// reference's semantics: its trainer runs all forwards and backwards of a
// mini-batch on unchanged weights and applies the queued updates afterwards
// (proj/src/nn.cpp:711-735), and the per-stream order of noise draws
// (forward, backward, update) is sample-major in both.
//
// The digital periphery (bias, activations, losses, the perfect_backward /
// perfect_update switches, weight-noise injection) runs on the host in double
// like the reference's; the analog tiles carry the O(N^2) work.  Host-side
// randomness (initialisation, datasets, shuffling, weight noise) uses
// RngStream, a restatement of proj/src/rng.cpp, so it reproduces the
// reference's draws bit for bit.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <fstream>
#include <limits>
#include <memory>
#include <numeric>
#include <optional>
#include <random>
#include <span>
#include <sstream>
#include <string>
#include <string_view>
#include <vector>

#include "tile.hpp"

namespace xbarsim_b200 {

// ---- proj/src/rng.cpp: named streams (splitmix64-derived seeds, mt19937_64,
// 53-bit uniforms, Box-Muller with a spare) ----
class RngStream {
public:
  explicit RngStream(uint64_t seed = 0) : seed_(seed), gen_(mix(seed)) {}
  RngStream derive(std::string_view name) const { return RngStream(mix(seed_ ^ fnv1a(name))); }
  RngStream derive(std::string_view name, uint64_t index) const {
    return RngStream(mix(mix(seed_ ^ fnv1a(name)) + index));
  }
  uint64_t base_seed() const { return seed_; }
  uint64_t next_u64() { return gen_(); }
  double uniform() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
  double gauss() {
    if (has_spare_) {
      has_spare_ = false;
      return spare_;
    }
    const double u1 = 1.0 - uniform(), u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1)), a = 2.0 * M_PI * u2;
    spare_ = r * std::sin(a);
    has_spare_ = true;
    return r * std::cos(a);
  }
  bool bernoulli(double p) { return p <= 0.0 ? false : (p >= 1.0 ? true : uniform() < p); }

private:
  static uint64_t fnv1a(std::string_view s) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (unsigned char c : s) {
      h ^= c;
      h *= 0x100000001b3ull;
    }
    return h;
  }
  static uint64_t mix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  uint64_t seed_;
  std::mt19937_64 gen_;
  bool has_spare_ = false;
  double spare_ = 0.0;
};

// ---- proj/include/xbarsim/nn.hpp:19-31 ----
enum class Activation { identity, tanh_act, relu, sigmoid };
enum class Loss { mse, cross_entropy };
enum class BiasMode { none, digital, analog };

struct HwAwareParams {
  bool perfect_backward = false;
  bool perfect_update = false;
  double weight_noise_sigma = 0.0;
};

// proj/src/nn.cpp:17-47
inline double apply_activation(Activation act, double z) {
  switch (act) {
  case Activation::identity:
    return z;
  case Activation::tanh_act:
    return std::tanh(z);
  case Activation::relu:
    return z > 0.0 ? z : 0.0;
  case Activation::sigmoid:
    return 1.0 / (1.0 + std::exp(-z));
  }
  return z;
}

inline double activation_grad(Activation act, double z) {
  switch (act) {
  case Activation::identity:
    return 1.0;
  case Activation::tanh_act: {
    const double t = std::tanh(z);
    return 1.0 - t * t;
  }
  case Activation::relu:
    return z > 0.0 ? 1.0 : 0.0;
  case Activation::sigmoid: {
    const double s = 1.0 / (1.0 + std::exp(-z));
    return s * (1.0 - s);
  }
  }
  return 1.0;
}

namespace nn_detail {
// y[b] = W x[b] / W^T x[b] in double (the perfect_* digital paths)
inline void matmul(const Matrix &w, const double *x, int B, double *y, bool transposed) {
  const int R = w.rows(), C = w.cols();
  for (int b = 0; b < B; ++b) {
    const double *xb = x + static_cast<size_t>(b) * (transposed ? R : C);
    double *yb = y + static_cast<size_t>(b) * (transposed ? C : R);
    if (!transposed) {
      for (int i = 0; i < R; ++i) {
        double acc = 0.0;
        for (int j = 0; j < C; ++j) acc += w(i, j) * xb[j];
        yb[i] = acc;
      }
    } else {
      for (int j = 0; j < C; ++j) yb[j] = 0.0;
      for (int i = 0; i < R; ++i)
        for (int j = 0; j < C; ++j) yb[j] += w(i, j) * xb[i];
    }
  }
}

inline Matrix noisy_copy(const Matrix &w, double sigma, RngStream &rng) { // nn.cpp:167-178
  Matrix n = w;
  for (int i = 0; i < n.rows(); ++i)
    for (int j = 0; j < n.cols(); ++j) n(i, j) += sigma * rng.gauss();
  return n;
}
} // namespace nn_detail

// ---- proj/include/xbarsim/nn.hpp:33-66: a layer hosting one analog tile ----
// Per-sample methods keep the reference's signatures; *_batch do B samples.
class LayerBase {
public:
  virtual ~LayerBase() = default;
  virtual int in_size() const = 0;
  virtual int out_size() const = 0;

  // B samples, row-major [B][in] -> [B][out]; cache = keep what backward needs
  virtual void forward_batch(const double *X, int B, double *Y, bool cache) = 0;
  // consumes the cached forward of the same B samples, queues their updates
  virtual void backward_batch(const double *G, int B, double *grad_in) = 0;
  virtual void forward_eval_batch(const double *X, int B, double *Y, double extra_weight_sigma,
                                  double output_scale) = 0;
  virtual void apply_updates(double lr, int batch_size) = 0;
  virtual void begin_minibatch(RngStream &rng) = 0;
  virtual void remove_weight_noise() = 0;
  virtual void end_minibatch() = 0;
  virtual TileBase &tile() = 0;
  virtual const TileBase &tile() const = 0;
  virtual std::unique_ptr<LayerBase> clone() const = 0;

  std::vector<double> forward(std::span<const double> x, bool cache) {
    std::vector<double> y(static_cast<size_t>(out_size()));
    forward_batch(x.data(), 1, y.data(), cache);
    return y;
  }
  std::vector<double> backward(std::span<const double> grad_out) {
    std::vector<double> g(static_cast<size_t>(in_size()));
    backward_batch(grad_out.data(), 1, g.data());
    return g;
  }
  std::vector<double> forward_eval(std::span<const double> x, double extra_weight_sigma,
                                   double output_scale) {
    std::vector<double> y(static_cast<size_t>(out_size()));
    forward_eval_batch(x.data(), 1, y.data(), extra_weight_sigma, output_scale);
    return y;
  }
};

// ---- proj/src/nn.cpp:52-208 ----
class AnalogDenseLayer : public LayerBase {
public:
  AnalogDenseLayer(std::unique_ptr<TileBase> tile, int in, int out, BiasMode bias_mode,
                   Activation act, HwAwareParams hw)
      : tile_(std::move(tile)), in_(in), out_(out), bias_mode_(bias_mode), act_(act), hw_(hw) {
    const int want_in = bias_mode_ == BiasMode::analog ? in_ + 1 : in_;
    if (tile_->d_out() != out_ || tile_->d_in() != want_in)
      throw Error("dense layer: tile shape " + std::to_string(tile_->d_out()) + "x" +
                  std::to_string(tile_->d_in()) + " does not match layer " +
                  std::to_string(out_) + "x" + std::to_string(want_in));
    if (bias_mode_ == BiasMode::digital) bias_.assign(static_cast<size_t>(out_), 0.0);
  }

  int in_size() const override { return in_; }
  int out_size() const override { return out_; }

  void forward_batch(const double *X, int B, double *Y, bool cache) override {
    std::vector<float> tin = tile_input(X, B);
    std::vector<float> z(static_cast<size_t>(B) * out_);
    tile_->forward_batch(tin.data(), B, z.data());
    std::vector<double> pre(z.size());
    for (int b = 0; b < B; ++b)
      for (int i = 0; i < out_; ++i) {
        const size_t k = static_cast<size_t>(b) * out_ + i;
        pre[k] = static_cast<double>(z[k]) + (bias_mode_ == BiasMode::digital ? bias_[i] : 0.0);
        Y[k] = apply_activation(act_, pre[k]);
      }
    if (cache) {
      cached_in_ = std::move(tin);
      cached_pre_ = std::move(pre);
      cached_b_ = B;
    }
  }

  void forward_eval_batch(const double *X, int B, double *Y, double extra,
                          double output_scale) override {
    std::vector<float> tin = tile_input(X, B);
    std::vector<float> z(static_cast<size_t>(B) * out_);
    tile_->forward_noisy_batch(tin.data(), B, z.data(), extra);
    for (int b = 0; b < B; ++b)
      for (int i = 0; i < out_; ++i) { // nn.cpp:96-110
        const size_t k = static_cast<size_t>(b) * out_ + i;
        double v = static_cast<double>(z[k]) * output_scale;
        if (bias_mode_ == BiasMode::digital) v += bias_[i];
        Y[k] = apply_activation(act_, v);
      }
  }

  void backward_batch(const double *G, int B, double *grad_in) override {
    if (cached_b_ == 0) throw Error("backward: no cached forward pass");
    if (B != cached_b_) throw Error("backward: gradient length mismatch");
    const int tin_n = tile_->d_in();
    std::vector<double> gz(static_cast<size_t>(B) * out_);
    for (size_t k = 0; k < gz.size(); ++k)
      gz[k] = G[k] * activation_grad(act_, cached_pre_[k]);
    std::vector<double> gi(static_cast<size_t>(B) * tin_n);
    if (hw_.perfect_backward) {
      nn_detail::matmul(tile_->get_weights(), gz.data(), B, gi.data(), true);
    } else {
      std::vector<float> gf(gz.begin(), gz.end()), gif(gi.size());
      tile_->backward_batch(gf.data(), B, gif.data());
      std::copy(gif.begin(), gif.end(), gi.begin());
    }
    for (int b = 0; b < B; ++b) // drop the constant-input column (nn.cpp:139-141)
      std::copy(gi.begin() + static_cast<size_t>(b) * tin_n,
                gi.begin() + static_cast<size_t>(b) * tin_n + in_,
                grad_in + static_cast<size_t>(b) * in_);
    q_in_.insert(q_in_.end(), cached_in_.begin(), cached_in_.end());
    q_gz_.insert(q_gz_.end(), gz.begin(), gz.end());
    cached_b_ = 0;
  }

  // nn.cpp:145-165: one batched pulsed update of every queued sample (or the
  // exact digital step under perfect_update), then the digital bias
  void apply_updates(double lr, int batch_size) override {
    const double inv_b = 1.0 / std::max(1, batch_size);
    const int n = static_cast<int>(q_gz_.size() / static_cast<size_t>(out_));
    const int tin_n = tile_->d_in();
    if (n > 0) {
      if (hw_.perfect_update) {
        Matrix w = tile_->get_weights();
        for (int s = 0; s < n; ++s)
          for (int i = 0; i < w.rows(); ++i)
            for (int j = 0; j < w.cols(); ++j)
              w(i, j) -= lr * inv_b * q_gz_[static_cast<size_t>(s) * out_ + i] *
                         q_in_[static_cast<size_t>(s) * tin_n + j];
        tile_->set_weights(w);
      } else {
        std::vector<float> d(q_gz_.size());
        for (size_t k = 0; k < d.size(); ++k) d[k] = static_cast<float>(-q_gz_[k] * inv_b);
        std::vector<double> l(static_cast<size_t>(n), lr);
        tile_->update_batch(q_in_.data(), d.data(), n, l.data());
      }
      if (bias_mode_ == BiasMode::digital)
        for (int s = 0; s < n; ++s)
          for (int i = 0; i < out_; ++i)
            bias_[i] -= lr * inv_b * q_gz_[static_cast<size_t>(s) * out_ + i];
    }
    q_in_.clear();
    q_gz_.clear();
  }

  void begin_minibatch(RngStream &rng) override {
    if (hw_.weight_noise_sigma > 0.0) {
      saved_ = tile_->get_weights();
      tile_->set_weights(nn_detail::noisy_copy(*saved_, hw_.weight_noise_sigma, rng));
    }
  }
  void remove_weight_noise() override {
    if (saved_) {
      tile_->set_weights(*saved_);
      saved_.reset();
    }
  }
  void end_minibatch() override { tile_->end_minibatch(); }

  TileBase &tile() override { return *tile_; }
  const TileBase &tile() const override { return *tile_; }
  std::unique_ptr<LayerBase> clone() const override {
    auto c = std::make_unique<AnalogDenseLayer>(tile_->clone(), in_, out_, bias_mode_, act_, hw_);
    c->bias_ = bias_;
    return c;
  }
  std::span<const double> bias() const { return bias_; }
  void set_bias(std::span<const double> b) {
    if (bias_mode_ != BiasMode::digital || static_cast<int>(b.size()) != out_)
      throw Error("set_bias: layer has no digital bias of that size");
    bias_.assign(b.begin(), b.end());
  }

private:
  std::vector<float> tile_input(const double *X, int B) const { // nn.cpp:68-74
    const int n = tile_->d_in();
    std::vector<float> v(static_cast<size_t>(B) * n);
    for (int b = 0; b < B; ++b) {
      for (int j = 0; j < in_; ++j)
        v[static_cast<size_t>(b) * n + j] = static_cast<float>(X[static_cast<size_t>(b) * in_ + j]);
      if (bias_mode_ == BiasMode::analog) v[static_cast<size_t>(b) * n + in_] = 1.0f;
    }
    return v;
  }

  std::unique_ptr<TileBase> tile_;
  int in_, out_;
  BiasMode bias_mode_;
  Activation act_;
  HwAwareParams hw_;
  std::vector<double> bias_;
  int cached_b_ = 0;
  std::vector<float> cached_in_;
  std::vector<double> cached_pre_;
  std::vector<float> q_in_;  // queued tile inputs [n][d_in]
  std::vector<double> q_gz_; // queued grad_z [n][out]
  std::optional<Matrix> saved_;
};

// ---- proj/src/nn.cpp:210-440: conv as one tile over unfolded patches; the
// patches of all samples of a batch go through the tile in one call, and the
// per-patch updates of a mini-batch are one weight-stationary update ----
class AnalogConv2DLayer : public LayerBase {
public:
  AnalogConv2DLayer(std::unique_ptr<TileBase> tile, int in_channels, int out_channels, int kernel,
                    int stride, int padding, int in_h, int in_w, BiasMode bias_mode,
                    Activation act, HwAwareParams hw)
      : tile_(std::move(tile)), cin_(in_channels), cout_(out_channels), k_(kernel),
        stride_(stride), pad_(padding), in_h_(in_h), in_w_(in_w), bias_mode_(bias_mode),
        act_(act), hw_(hw) {
    if (k_ < 1 || stride_ < 1 || pad_ < 0) throw Error("conv layer: invalid kernel/stride/padding");
    if (bias_mode_ == BiasMode::analog) throw Error("conv layer: analog bias not supported");
    out_h_ = (in_h_ + 2 * pad_ - k_) / stride_ + 1;
    out_w_ = (in_w_ + 2 * pad_ - k_) / stride_ + 1;
    if (out_h_ < 1 || out_w_ < 1) throw Error("conv layer: kernel does not fit the input");
    if (tile_->d_out() != cout_ || tile_->d_in() != cin_ * k_ * k_)
      throw Error("conv layer: tile shape must be out_channels x (in_channels*k*k)");
    if (bias_mode_ == BiasMode::digital) bias_.assign(static_cast<size_t>(cout_), 0.0);
  }

  int in_size() const override { return cin_ * in_h_ * in_w_; }
  int out_size() const override { return cout_ * out_h_ * out_w_; }
  int out_h() const { return out_h_; }
  int out_w() const { return out_w_; }

  // nn.cpp:235-256
  std::vector<double> unfold_patch(std::span<const double> x, int oy, int ox) const {
    std::vector<double> p(static_cast<size_t>(cin_ * k_ * k_), 0.0);
    for (int c = 0; c < cin_; ++c)
      for (int ky = 0; ky < k_; ++ky) {
        const int iy = oy * stride_ + ky - pad_;
        if (iy < 0 || iy >= in_h_) continue;
        for (int kx = 0; kx < k_; ++kx) {
          const int ix = ox * stride_ + kx - pad_;
          if (ix < 0 || ix >= in_w_) continue;
          p[static_cast<size_t>((c * k_ + ky) * k_ + kx)] = x[static_cast<size_t>((c * in_h_ + iy) * in_w_ + ix)];
        }
      }
    return p;
  }

  void forward_batch(const double *X, int B, double *Y, bool cache) override {
    const int P = out_h_ * out_w_;
    std::vector<float> patches = unfold_all(X, B);
    std::vector<float> cols(static_cast<size_t>(B) * P * cout_);
    tile_->forward_batch(patches.data(), B * P, cols.data());
    std::vector<double> pre(static_cast<size_t>(B) * out_size());
    scatter(cols, B, 1.0, pre.data());
    for (size_t k = 0; k < pre.size(); ++k) Y[k] = apply_activation(act_, pre[k]);
    if (cache) {
      cached_patches_ = std::move(patches);
      cached_pre_ = std::move(pre);
      cached_b_ = B;
    }
  }

  void forward_eval_batch(const double *X, int B, double *Y, double extra,
                          double output_scale) override {
    const int P = out_h_ * out_w_;
    std::vector<float> patches = unfold_all(X, B);
    std::vector<float> cols(static_cast<size_t>(B) * P * cout_);
    tile_->forward_noisy_batch(patches.data(), B * P, cols.data(), extra);
    scatter(cols, B, output_scale, Y);
    for (int k = 0; k < B * out_size(); ++k) Y[k] = apply_activation(act_, Y[k]);
  }

  // nn.cpp:310-364
  void backward_batch(const double *G, int B, double *grad_in) override {
    if (cached_b_ == 0) throw Error("backward: no cached forward pass");
    if (B != cached_b_) throw Error("conv backward: gradient length mismatch");
    const int P = out_h_ * out_w_, KK = cin_ * k_ * k_;
    std::vector<double> gcol(static_cast<size_t>(B) * P * cout_);
    for (int b = 0; b < B; ++b)
      for (int p = 0; p < P; ++p)
        for (int c = 0; c < cout_; ++c) {
          const size_t pos = static_cast<size_t>(b) * out_size() + static_cast<size_t>(c) * P + p;
          gcol[(static_cast<size_t>(b) * P + p) * cout_ + c] =
              G[pos] * activation_grad(act_, cached_pre_[pos]);
        }
    std::vector<double> gpatch(static_cast<size_t>(B) * P * KK);
    if (hw_.perfect_backward) {
      nn_detail::matmul(tile_->get_weights(), gcol.data(), B * P, gpatch.data(), true);
    } else {
      std::vector<float> gf(gcol.begin(), gcol.end()), pf(gpatch.size());
      tile_->backward_batch(gf.data(), B * P, pf.data());
      std::copy(pf.begin(), pf.end(), gpatch.begin());
    }
    std::fill(grad_in, grad_in + static_cast<size_t>(B) * in_size(), 0.0);
    for (int b = 0; b < B; ++b) // fold the patch gradients back onto the input grid
      for (int oy = 0; oy < out_h_; ++oy)
        for (int ox = 0; ox < out_w_; ++ox) {
          const double *gp = gpatch.data() + (static_cast<size_t>(b) * P + oy * out_w_ + ox) * KK;
          double *gi = grad_in + static_cast<size_t>(b) * in_size();
          for (int c = 0; c < cin_; ++c)
            for (int ky = 0; ky < k_; ++ky) {
              const int iy = oy * stride_ + ky - pad_;
              if (iy < 0 || iy >= in_h_) continue;
              for (int kx = 0; kx < k_; ++kx) {
                const int ix = ox * stride_ + kx - pad_;
                if (ix < 0 || ix >= in_w_) continue;
                gi[(c * in_h_ + iy) * in_w_ + ix] += gp[(c * k_ + ky) * k_ + kx];
              }
            }
        }
    q_patch_.insert(q_patch_.end(), cached_patches_.begin(), cached_patches_.end());
    q_gcol_.insert(q_gcol_.end(), gcol.begin(), gcol.end());
    cached_b_ = 0;
    cached_patches_.clear();
  }

  // nn.cpp:366-398: the per-patch updates of the mini-batch as ONE batched
  // update, samples and patches in the reference's queue order
  void apply_updates(double lr, int batch_size) override {
    const double inv_b = 1.0 / std::max(1, batch_size);
    const int KK = cin_ * k_ * k_;
    const int n = static_cast<int>(q_gcol_.size() / static_cast<size_t>(cout_));
    if (n > 0) {
      if (hw_.perfect_update) {
        Matrix w = tile_->get_weights();
        for (int s = 0; s < n; ++s)
          for (int i = 0; i < w.rows(); ++i)
            for (int j = 0; j < w.cols(); ++j)
              w(i, j) -= lr * inv_b * q_gcol_[static_cast<size_t>(s) * cout_ + i] *
                         q_patch_[static_cast<size_t>(s) * KK + j];
        tile_->set_weights(w);
      } else {
        std::vector<float> d(q_gcol_.size());
        for (size_t k = 0; k < d.size(); ++k) d[k] = static_cast<float>(-q_gcol_[k] * inv_b);
        std::vector<double> l(static_cast<size_t>(n), lr);
        tile_->update_batch(q_patch_.data(), d.data(), n, l.data());
      }
      if (bias_mode_ == BiasMode::digital)
        for (int s = 0; s < n; ++s)
          for (int c = 0; c < cout_; ++c)
            bias_[c] -= lr * inv_b * q_gcol_[static_cast<size_t>(s) * cout_ + c];
    }
    q_patch_.clear();
    q_gcol_.clear();
  }

  void begin_minibatch(RngStream &rng) override {
    if (hw_.weight_noise_sigma > 0.0) {
      saved_ = tile_->get_weights();
      tile_->set_weights(nn_detail::noisy_copy(*saved_, hw_.weight_noise_sigma, rng));
    }
  }
  void remove_weight_noise() override {
    if (saved_) {
      tile_->set_weights(*saved_);
      saved_.reset();
    }
  }
  void end_minibatch() override { tile_->end_minibatch(); }
  TileBase &tile() override { return *tile_; }
  const TileBase &tile() const override { return *tile_; }
  std::unique_ptr<LayerBase> clone() const override {
    auto c = std::make_unique<AnalogConv2DLayer>(tile_->clone(), cin_, cout_, k_, stride_, pad_,
                                                 in_h_, in_w_, bias_mode_, act_, hw_);
    c->bias_ = bias_;
    return c;
  }

private:
  std::vector<float> unfold_all(const double *X, int B) const {
    const int P = out_h_ * out_w_, KK = cin_ * k_ * k_;
    std::vector<float> out(static_cast<size_t>(B) * P * KK);
    for (int b = 0; b < B; ++b) {
      std::span<const double> x(X + static_cast<size_t>(b) * in_size(),
                                static_cast<size_t>(in_size()));
      for (int oy = 0; oy < out_h_; ++oy)
        for (int ox = 0; ox < out_w_; ++ox) {
          const std::vector<double> p = unfold_patch(x, oy, ox);
          std::copy(p.begin(), p.end(),
                    out.begin() + (static_cast<size_t>(b) * P + oy * out_w_ + ox) * KK);
        }
    }
    return out;
  }
  // columns [b][p][c] -> channel-major [b][c][oy][ox], times scale, plus bias
  void scatter(const std::vector<float> &cols, int B, double scale, double *z) const {
    const int P = out_h_ * out_w_;
    for (int b = 0; b < B; ++b)
      for (int p = 0; p < P; ++p)
        for (int c = 0; c < cout_; ++c) {
          double v = static_cast<double>(cols[(static_cast<size_t>(b) * P + p) * cout_ + c]) * scale;
          if (bias_mode_ == BiasMode::digital) v += bias_[c];
          z[static_cast<size_t>(b) * out_size() + static_cast<size_t>(c) * P + p] = v;
        }
  }

  std::unique_ptr<TileBase> tile_;
  int cin_, cout_, k_, stride_, pad_, in_h_, in_w_;
  int out_h_ = 0, out_w_ = 0;
  BiasMode bias_mode_;
  Activation act_;
  HwAwareParams hw_;
  std::vector<double> bias_;
  int cached_b_ = 0;
  std::vector<float> cached_patches_;
  std::vector<double> cached_pre_;
  std::vector<float> q_patch_;
  std::vector<double> q_gcol_;
  std::optional<Matrix> saved_;
};

// ---- proj/src/nn.cpp:442-495 ----
class Network {
public:
  Network() = default;
  Network(const Network &o) {
    for (const auto &l : o.layers_) layers_.push_back(l->clone());
  }
  Network &operator=(const Network &o) {
    if (this != &o) {
      Network tmp(o);
      layers_ = std::move(tmp.layers_);
    }
    return *this;
  }
  Network(Network &&) = default;
  Network &operator=(Network &&) = default;

  void add(std::unique_ptr<LayerBase> layer) {
    if (!layers_.empty() && layers_.back()->out_size() != layer->in_size())
      throw Error("network: layer input " + std::to_string(layer->in_size()) +
                  " does not match previous output " + std::to_string(layers_.back()->out_size()));
    layers_.push_back(std::move(layer));
  }
  int n_layers() const { return static_cast<int>(layers_.size()); }
  LayerBase &layer(int i) { return *layers_[static_cast<size_t>(i)]; }
  const LayerBase &layer(int i) const { return *layers_[static_cast<size_t>(i)]; }
  int in_size() const { return layers_.empty() ? 0 : layers_.front()->in_size(); }
  int out_size() const { return layers_.empty() ? 0 : layers_.back()->out_size(); }

  std::vector<double> forward_batch(const double *X, int B, bool cache) {
    std::vector<double> v(X, X + static_cast<size_t>(B) * in_size());
    for (auto &l : layers_) {
      std::vector<double> y(static_cast<size_t>(B) * l->out_size());
      l->forward_batch(v.data(), B, y.data(), cache);
      v = std::move(y);
    }
    return v;
  }
  std::vector<double> backward_batch(const double *G, int B) {
    std::vector<double> g(G, G + static_cast<size_t>(B) * out_size());
    for (auto it = layers_.rbegin(); it != layers_.rend(); ++it) {
      std::vector<double> gi(static_cast<size_t>(B) * (*it)->in_size());
      (*it)->backward_batch(g.data(), B, gi.data());
      g = std::move(gi);
    }
    return g;
  }
  std::vector<double> forward(std::span<const double> x, bool cache) {
    return forward_batch(x.data(), 1, cache);
  }
  std::vector<double> backward(std::span<const double> g) { return backward_batch(g.data(), 1); }
  void apply_updates(double lr, int batch_size) {
    for (auto &l : layers_) l->apply_updates(lr, batch_size);
  }
  void begin_minibatch(RngStream &rng) {
    for (auto &l : layers_) l->begin_minibatch(rng);
  }
  void remove_weight_noise() {
    for (auto &l : layers_) l->remove_weight_noise();
  }
  void end_minibatch() {
    for (auto &l : layers_) l->end_minibatch();
  }
  std::vector<double> forward_eval_batch(const double *X, int B, double extra_weight_sigma,
                                         std::span<const double> output_scales) {
    std::vector<double> v(X, X + static_cast<size_t>(B) * in_size());
    for (size_t i = 0; i < layers_.size(); ++i) {
      const double scale = output_scales.empty() ? 1.0 : output_scales[i];
      std::vector<double> y(static_cast<size_t>(B) * layers_[i]->out_size());
      layers_[i]->forward_eval_batch(v.data(), B, y.data(), extra_weight_sigma, scale);
      v = std::move(y);
    }
    return v;
  }
  std::vector<double> forward_eval(std::span<const double> x, double extra_weight_sigma,
                                   std::span<const double> output_scales) {
    return forward_eval_batch(x.data(), 1, extra_weight_sigma, output_scales);
  }

private:
  std::vector<std::unique_ptr<LayerBase>> layers_;
};

// proj/src/nn.cpp:497-512
inline void initialize_network(Network &net, uint64_t seed) {
  RngStream rng(seed);
  for (int l = 0; l < net.n_layers(); ++l) {
    RngStream stream = rng.derive("init", static_cast<uint64_t>(l));
    TileBase &tile = net.layer(l).tile();
    Matrix w(tile.d_out(), tile.d_in());
    const double scale = 1.0 / std::sqrt(static_cast<double>(tile.d_in()));
    for (int i = 0; i < w.rows(); ++i)
      for (int j = 0; j < w.cols(); ++j) w(i, j) = scale * (2.0 * stream.uniform() - 1.0);
    tile.set_weights(w);
  }
}

// ---- losses, proj/src/nn.cpp:517-560 ----
struct LossGrad {
  double loss = 0.0;
  std::vector<double> grad;
};

inline LossGrad loss_mse(std::span<const double> pred, std::span<const double> target) {
  if (pred.size() != target.size()) throw Error("mse: prediction/target size mismatch");
  LossGrad out;
  out.grad.resize(pred.size());
  const double inv_n = 1.0 / static_cast<double>(pred.size());
  for (size_t i = 0; i < pred.size(); ++i) {
    const double e = pred[i] - target[i];
    out.loss += e * e * inv_n;
    out.grad[i] = 2.0 * e * inv_n;
  }
  return out;
}

inline LossGrad loss_cross_entropy(std::span<const double> logits, int label) {
  if (label < 0 || label >= static_cast<int>(logits.size()))
    throw Error("cross_entropy: label out of range");
  LossGrad out;
  out.grad.resize(logits.size());
  double zmax = -std::numeric_limits<double>::infinity();
  for (double z : logits) zmax = std::max(zmax, z);
  double denom = 0.0;
  for (double z : logits) denom += std::exp(z - zmax);
  for (size_t i = 0; i < logits.size(); ++i) {
    const double p = std::exp(logits[i] - zmax) / denom;
    out.grad[i] = p - (static_cast<int>(i) == label ? 1.0 : 0.0);
    if (static_cast<int>(i) == label) out.loss = -(logits[i] - zmax - std::log(denom));
  }
  return out;
}

// ---- datasets, proj/include/xbarsim/nn.hpp:200-225, proj/src/nn.cpp:565-680 ----
struct Dataset {
  int n_features = 0;
  int n_outputs = 0;
  bool classification = true;
  std::vector<std::vector<double>> inputs;
  std::vector<int> labels;
  std::vector<std::vector<double>> targets;
  size_t size() const { return inputs.size(); }
  std::vector<double> target_of(size_t idx) const {
    if (classification) {
      std::vector<double> t(static_cast<size_t>(n_outputs), 0.0);
      t[static_cast<size_t>(labels[idx])] = 1.0;
      return t;
    }
    return targets[idx];
  }
};

inline Dataset make_blobs(int n, int features, int classes, double spread, uint64_t seed,
                          uint64_t sample_salt = 0) {
  RngStream center_rng = RngStream(seed).derive("blob_centers");
  RngStream sample_rng = RngStream(seed).derive("blob_samples", sample_salt);
  Dataset d;
  d.n_features = features;
  d.n_outputs = classes;
  d.classification = true;
  std::vector<std::vector<double>> centers(static_cast<size_t>(classes),
                                           std::vector<double>(static_cast<size_t>(features)));
  for (auto &c : centers) {
    double norm = 0.0;
    for (double &v : c) {
      v = center_rng.gauss();
      norm += v * v;
    }
    norm = std::sqrt(norm);
    for (double &v : c) v /= (norm > 0.0 ? norm : 1.0);
  }
  for (int s = 0; s < n; ++s) {
    const int c = s % classes;
    std::vector<double> x(static_cast<size_t>(features));
    for (int f = 0; f < features; ++f)
      x[static_cast<size_t>(f)] = centers[static_cast<size_t>(c)][static_cast<size_t>(f)] +
                                  spread * sample_rng.gauss();
    d.inputs.push_back(std::move(x));
    d.labels.push_back(c);
  }
  return d;
}

inline Dataset make_regression(int n, int features, int outputs, double noise, uint64_t seed,
                               uint64_t sample_salt = 0) {
  RngStream model_rng = RngStream(seed).derive("regression_model");
  RngStream sample_rng = RngStream(seed).derive("regression_samples", sample_salt);
  Dataset d;
  d.n_features = features;
  d.n_outputs = outputs;
  d.classification = false;
  Matrix a(outputs, features);
  for (int i = 0; i < outputs; ++i)
    for (int j = 0; j < features; ++j) a(i, j) = 2.0 * model_rng.uniform() - 1.0;
  for (int s = 0; s < n; ++s) {
    std::vector<double> x(static_cast<size_t>(features));
    for (double &v : x) v = 2.0 * sample_rng.uniform() - 1.0;
    std::vector<double> t(static_cast<size_t>(outputs), 0.0);
    for (int i = 0; i < outputs; ++i)
      for (int j = 0; j < features; ++j) t[static_cast<size_t>(i)] += a(i, j) * x[static_cast<size_t>(j)];
    for (double &v : t) v += noise * sample_rng.gauss();
    d.inputs.push_back(std::move(x));
    d.targets.push_back(std::move(t));
  }
  return d;
}

inline Dataset load_csv_dataset(const std::string &path, bool classification) {
  std::ifstream in(path);
  if (!in) throw Error("dataset: cannot open '" + path + "'");
  Dataset d;
  d.classification = classification;
  std::string line;
  int max_label = -1;
  while (std::getline(in, line)) {
    if (line.empty() || line[0] == '#') continue;
    std::vector<double> row;
    std::stringstream ss(line);
    std::string cell;
    while (std::getline(ss, cell, ',')) row.push_back(std::stod(cell));
    if (row.size() < 2) throw Error("dataset: row with fewer than 2 columns in '" + path + "'");
    if (d.n_features == 0)
      d.n_features = static_cast<int>(row.size()) - 1;
    else if (static_cast<int>(row.size()) - 1 != d.n_features)
      throw Error("dataset: inconsistent column count in '" + path + "'");
    const double last = row.back();
    row.pop_back();
    d.inputs.push_back(std::move(row));
    if (classification) {
      const int label = static_cast<int>(std::lround(last));
      d.labels.push_back(label);
      max_label = std::max(max_label, label);
    } else {
      d.targets.push_back({last});
    }
  }
  d.n_outputs = classification ? max_label + 1 : 1;
  return d;
}

// ---- trainer, proj/include/xbarsim/nn.hpp:227-246, proj/src/nn.cpp:686-760 ----
struct TrainConfig {
  Loss loss = Loss::mse;
  double lr = 0.1;
  double lr_decay = 1.0;
  int epochs = 30;
  int batch_size = 10;
  uint64_t seed = 1234;
};

struct EpochStats {
  int epoch = 0;
  double loss = 0.0;
  double accuracy = 0.0;
};

// The reference's loop with each mini-batch as one batched pass per layer:
// forward(all samples, cache) -> per-sample loss -> backward(all samples) ->
// remove weight noise -> one batched update per layer -> end_minibatch.
inline std::vector<EpochStats> train(Network &net, const Dataset &data, const TrainConfig &cfg) {
  if (data.size() == 0) throw Error("train: empty dataset");
  if (cfg.epochs < 0 || cfg.batch_size < 1) throw Error("train: invalid epochs/batch_size");
  if (cfg.loss == Loss::cross_entropy && !data.classification)
    throw Error("train: cross_entropy needs a classification dataset");
  RngStream shuffle_rng = RngStream(cfg.seed).derive("shuffle");
  RngStream wnoise_rng = RngStream(cfg.seed).derive("weight_noise");
  std::vector<size_t> order(data.size());
  std::iota(order.begin(), order.end(), size_t{0});
  std::vector<EpochStats> history;
  double lr = cfg.lr;
  const int nin = net.in_size(), nout = net.out_size();
  for (int epoch = 0; epoch < cfg.epochs; ++epoch) {
    for (size_t i = order.size(); i > 1; --i) { // Fisher-Yates on the shuffle stream
      const size_t j = static_cast<size_t>(shuffle_rng.uniform() * static_cast<double>(i));
      std::swap(order[i - 1], order[std::min(j, i - 1)]);
    }
    double loss_sum = 0.0;
    long correct = 0;
    for (size_t start = 0; start < order.size(); start += static_cast<size_t>(cfg.batch_size)) {
      const size_t stop = std::min(order.size(), start + static_cast<size_t>(cfg.batch_size));
      const int B = static_cast<int>(stop - start);
      net.begin_minibatch(wnoise_rng);
      std::vector<double> X(static_cast<size_t>(B) * nin);
      for (int b = 0; b < B; ++b) {
        const auto &x = data.inputs[order[start + static_cast<size_t>(b)]];
        std::copy(x.begin(), x.end(), X.begin() + static_cast<size_t>(b) * nin);
      }
      const std::vector<double> Y = net.forward_batch(X.data(), B, true);
      std::vector<double> G(static_cast<size_t>(B) * nout);
      for (int b = 0; b < B; ++b) {
        const size_t idx = order[start + static_cast<size_t>(b)];
        std::span<const double> y(Y.data() + static_cast<size_t>(b) * nout, static_cast<size_t>(nout));
        LossGrad lg = cfg.loss == Loss::cross_entropy ? loss_cross_entropy(y, data.labels[idx])
                                                      : loss_mse(y, data.target_of(idx));
        loss_sum += lg.loss;
        if (data.classification) {
          const auto arg = std::distance(y.begin(), std::max_element(y.begin(), y.end()));
          correct += (arg == data.labels[idx]) ? 1 : 0;
        }
        std::copy(lg.grad.begin(), lg.grad.end(), G.begin() + static_cast<size_t>(b) * nout);
      }
      net.backward_batch(G.data(), B);
      net.remove_weight_noise();
      net.apply_updates(lr, B);
      net.end_minibatch();
    }
    EpochStats st;
    st.epoch = epoch;
    st.loss = loss_sum / static_cast<double>(data.size());
    st.accuracy = data.classification
                      ? static_cast<double>(correct) / static_cast<double>(data.size())
                      : std::numeric_limits<double>::quiet_NaN();
    history.push_back(st);
    lr *= cfg.lr_decay;
  }
  return history;
}

inline double evaluate_accuracy(Network &net, const Dataset &data) {
  const int nin = net.in_size(), nout = net.out_size();
  const int B = static_cast<int>(data.size());
  std::vector<double> X(static_cast<size_t>(B) * nin);
  for (int b = 0; b < B; ++b)
    std::copy(data.inputs[static_cast<size_t>(b)].begin(), data.inputs[static_cast<size_t>(b)].end(),
              X.begin() + static_cast<size_t>(b) * nin);
  const std::vector<double> Y = net.forward_batch(X.data(), B, false);
  long correct = 0;
  for (int b = 0; b < B; ++b) {
    auto first = Y.begin() + static_cast<size_t>(b) * nout;
    correct += (std::distance(first, std::max_element(first, first + nout)) ==
                data.labels[static_cast<size_t>(b)]);
  }
  return static_cast<double>(correct) / static_cast<double>(B);
}

inline double evaluate_mse(Network &net, const Dataset &data) {
  const int nin = net.in_size(), nout = net.out_size();
  const int B = static_cast<int>(data.size());
  std::vector<double> X(static_cast<size_t>(B) * nin);
  for (int b = 0; b < B; ++b)
    std::copy(data.inputs[static_cast<size_t>(b)].begin(), data.inputs[static_cast<size_t>(b)].end(),
              X.begin() + static_cast<size_t>(b) * nin);
  const std::vector<double> Y = net.forward_batch(X.data(), B, false);
  double acc = 0.0;
  for (int b = 0; b < B; ++b)
    acc += loss_mse(std::span<const double>(Y.data() + static_cast<size_t>(b) * nout,
                                            static_cast<size_t>(nout)),
                    data.target_of(static_cast<size_t>(b)))
               .loss;
  return acc / static_cast<double>(B);
}

} // namespace xbarsim_b200
