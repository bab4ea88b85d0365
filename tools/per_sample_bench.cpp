// Per-sample drop-in path through the C++ mirror of the reference API
// (include/xbarsim_b200/tile.hpp): TileBase::forward(x) one sample per call
// (host vectors in, host vector out -- what proj/src/nn.cpp calls per sample)
// and TileBase::update(x, d, lr) per sample (queued; the queue is applied as
// one weight-stationary batched update when the weights are next read, SURVEY
// section 8b).  4096 x 4096 reram_sb tile, default IO.  Prints one JSON line:
//   tools/per_sample_bench [--n 4096] [--samples 256]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "xbarsim_b200/tile.hpp"

using namespace xbarsim_b200;
using clk = std::chrono::steady_clock;

int main(int argc, char **argv) {
  int n = 4096, samples = 256;
  for (int i = 1; i + 1 < argc; i += 2) {
    if (!std::strcmp(argv[i], "--n")) n = std::atoi(argv[i + 1]);
    if (!std::strcmp(argv[i], "--samples")) samples = std::atoi(argv[i + 1]);
  }
  TileSettings s;
  s.device = device_preset("reram_sb");
  AnalogTile t(n, n, s, 1234);
  std::mt19937_64 g(7);
  std::uniform_real_distribution<double> u(-1.0, 1.0), uw(-0.1, 0.1);
  Matrix w0(n, n);
  for (size_t k = 0; k < w0.size(); ++k) w0.data()[k] = uw(g);
  t.set_weights(w0);
  std::vector<std::vector<double>> xs(samples, std::vector<double>(n)),
      ds(samples, std::vector<double>(n));
  for (auto &v : xs)
    for (double &e : v) e = u(g);
  for (auto &v : ds)
    for (double &e : v) e = u(g);
  for (int k = 0; k < 8; ++k) (void)t.forward(xs[k]); // warm
  auto t0 = clk::now();
  double acc = 0.0;
  for (int k = 0; k < samples; ++k) acc += t.forward(xs[k])[0];
  const double fwd_s = std::chrono::duration<double>(clk::now() - t0).count();
  for (int k = 0; k < samples; ++k) t.update(xs[k], ds[k], 0.01);
  (void)t.forward(xs[0]); // warm: the next read applies the queue
  t0 = clk::now();
  for (int k = 0; k < samples; ++k) t.update(xs[k], ds[k], 0.01);
  acc += t.forward(xs[0])[0]; // applies the queued samples (one batched update), then reads
  const double upd_s =
      std::chrono::duration<double>(clk::now() - t0).count() - fwd_s / samples;
  const double cells = (double)n * n;
  std::printf("{\"n\": %d, \"samples\": %d, \"forward_us_per_sample\": %.3f, "
              "\"forward_samples_per_s\": %.1f, \"update_us_per_sample\": %.3f, "
              "\"update_cell_updates_per_s\": %.4g, \"checksum\": %.6g, "
              "\"api\": \"xbarsim_b200::AnalogTile (TileBase) forward(x) / update(x, d, lr), "
              "host std::vector<double> per sample; the queued updates are applied by the next "
              "forward (its own time subtracted)\"}\n",
              n, samples, fwd_s / samples * 1e6, samples / fwd_s, upd_s / samples * 1e6,
              cells * samples / upd_s, acc);
  return 0;
}
