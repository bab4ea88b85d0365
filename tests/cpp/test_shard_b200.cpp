// C++ row-sharded tile (include/xbarsim_b200/tile.hpp: Comm, RowShardedTile)
// on one GPU: P ranks of a loopback group, one std::thread per rank (as one
// process per GPU would drive them).  update and forward (bound management
// on) must equal the unsharded AnalogTile bit for bit; the backward within
// one ADC LSB (fp32 order of the cross-rank sum).  Run by
// tests/test_gpu_cpp.py; exits non-zero on failure.
#include <cmath>
#include <cstdio>
#include <random>
#include <thread>
#include <vector>

#include "xbarsim_b200/tile.hpp"

using namespace xbarsim_b200;

static int run(int P, int R, int C, int B, MvmPrecision prec) {
  TileSettings s;
  s.device = device_preset("reram_sb");
  s.forward_io.bound_management = BoundManagement::iterative;
  s.forward_io.sigma_w = 0.01;
  s.mvm_precision = prec;
  std::mt19937_64 g(17);
  std::uniform_real_distribution<float> uw(-0.5f, 0.5f), u(-1.f, 1.f);
  std::vector<float> W((size_t)R * C), X((size_t)B * C), D((size_t)B * R);
  for (auto &v : W) v = uw(g);
  for (auto &v : X) v = u(g);
  for (auto &v : D) v = u(g);

  AnalogTile full(R, C, s, 42);
  Matrix Wm(R, C);
  for (size_t k = 0; k < W.size(); ++k) Wm.data()[k] = W[k];
  full.set_weights(Wm);
  std::vector<float> Yf((size_t)B * R), Gf((size_t)B * C), Yf2((size_t)B * R);
  full.forward_batch(X.data(), B, Yf.data());
  full.backward_batch(D.data(), B, Gf.data());
  full.update_batch(X.data(), D.data(), B, nullptr);
  full.forward_batch(X.data(), B, Yf2.data());
  Matrix Wf = full.get_weights();

  std::vector<Comm> comms = Comm::local(P);
  std::vector<std::vector<float>> Y(P), G(P), Y2(P), Wl(P);
  std::vector<std::pair<int, int>> rows(P);
  std::vector<std::string> err(P);
  std::vector<std::thread> th;
  for (int q = 0; q < P; ++q)
    th.emplace_back([&, q] {
      try {
        RowShardedTile t(R, C, s, 42, comms[q]);
        const int r0 = t.row_begin(), n = t.local_rows();
        rows[q] = {r0, n};
        t.set_weights(W.data() + (size_t)r0 * C);
        std::vector<float> Dl((size_t)B * n);
        for (int b = 0; b < B; ++b)
          for (int i = 0; i < n; ++i) Dl[(size_t)b * n + i] = D[(size_t)b * R + r0 + i];
        Y[q].resize((size_t)B * n);
        G[q].resize((size_t)B * C);
        Y2[q].resize((size_t)B * n);
        t.forward_batch(X.data(), B, Y[q].data());
        t.backward_batch(Dl.data(), B, G[q].data());
        t.update_batch(X.data(), Dl.data(), B, nullptr);
        t.forward_batch(X.data(), B, Y2[q].data());
        Wl[q] = t.get_weights();
      } catch (const std::exception &e) {
        err[q] = e.what();
      }
    });
  for (auto &t : th) t.join();
  int fail = 0;
  for (int q = 0; q < P; ++q)
    if (!err[q].empty()) {
      std::printf("  rank %d: %s\n", q, err[q].c_str());
      ++fail;
    }
  if (fail) return fail;
  long ydiff = 0, wdiff = 0, gbad = 0, goff = 0;
  for (int q = 0; q < P; ++q) {
    const int r0 = rows[q].first, n = rows[q].second;
    for (int b = 0; b < B; ++b)
      for (int i = 0; i < n; ++i) {
        ydiff += Y[q][(size_t)b * n + i] != Yf[(size_t)b * R + r0 + i];
        ydiff += Y2[q][(size_t)b * n + i] != Yf2[(size_t)b * R + r0 + i];
      }
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < C; ++j) wdiff += Wl[q][(size_t)i * C + j] != (float)Wf(r0 + i, j);
    for (int b = 0; b < B; ++b) {
      float dm = 0.f;
      for (int i = 0; i < R; ++i) dm = std::max(dm, std::fabs(D[(size_t)b * R + i]));
      const double lsb = 2 * 12.0 / 512 * dm;
      for (int j = 0; j < C; ++j) {
        const double d = std::fabs((double)G[q][(size_t)b * C + j] - Gf[(size_t)b * C + j]);
        gbad += d > lsb * 1.001 + 1e-6;
        goff += d > 1e-6;
      }
    }
  }
  const bool ok = ydiff == 0 && wdiff == 0 && gbad == 0 && goff < 0.02 * P * B * C;
  std::printf("%s P=%d %dx%d B=%d prec=%d: forward/update mismatches %ld/%ld, backward >1 LSB %ld, off-grid %ld\n",
              ok ? "ok  " : "FAIL", P, R, C, B, (int)prec, ydiff, wdiff, gbad, goff);
  return ok ? 0 : 1;
}

int main() {
  int fail = 0;
  fail += run(2, 1024, 512, 256, MvmPrecision::tf32);
  fail += run(4, 700, 300, 40, MvmPrecision::tf32x3);
  fail += run(3, 96, 64, 12, MvmPrecision::fp32);
  std::printf("%s\n", fail ? "FAILED" : "all sharded cases passed");
  return fail ? 1 : 0;
}
