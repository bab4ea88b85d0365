// matvec_bench_b200 -- the reference CLI's `matvec-bench` subcommand
// (proj/tools/xbarsim_main.cpp:162-212) on the B200 tile.
//
//   matvec_bench_b200 [--size 256] [--reps 100] [--out .] [--seed 1234] [--batched]
//
// Same workload and output file as the reference: an ideal-device size x size
// tile with W ~ 0.1 N(0,1) and x ~ N(0,1) drawn from RngStream(seed) "bench",
// `reps` analog forwards timed against `reps` digital mat-vecs, written to
// <out>/matvec_bench.csv (timings as '#' comments, the body = size, reps and
// both checksums).  --batched issues the reps as ONE batched forward (the
// B200 path's natural form) instead of reps single-sample calls.
#include <charconv>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <sys/stat.h>
#include <vector>

#include "xbarsim_b200/nn.hpp"

using namespace xbarsim_b200;

static std::string fmt_double(double v) { // proj/include/xbarsim/csv.hpp:18-22
  char buf[32];
  auto res = std::to_chars(buf, buf + sizeof(buf), v);
  return std::string(buf, res.ptr);
}

int main(int argc, char **argv) {
  int size = 256, reps = 100;
  uint64_t seed = 1234;
  std::string out_dir = ".";
  bool batched = false;
  for (int a = 1; a < argc; ++a) {
    const std::string k = argv[a];
    auto val = [&]() -> std::string {
      if (a + 1 >= argc) throw Error("missing value for " + k);
      return argv[++a];
    };
    try {
      if (k == "--size") size = std::stoi(val());
      else if (k == "--reps") reps = std::stoi(val());
      else if (k == "--seed") seed = std::stoull(val());
      else if (k == "--out") out_dir = val();
      else if (k == "--batched") batched = true;
      else throw Error("unknown option " + k);
    } catch (const std::exception &e) {
      std::fprintf(stderr, "error: %s\n", e.what());
      return 1;
    }
  }
  try {
    mkdir(out_dir.c_str(), 0755);
    TileSettings settings;
    settings.device = device_preset("ideal");
    AnalogTile tile(size, size, settings, seed);
    RngStream rng = RngStream(seed).derive("bench");
    Matrix w(size, size);
    std::vector<double> x(static_cast<size_t>(size));
    for (int i = 0; i < size; ++i) {
      for (int j = 0; j < size; ++j) w(i, j) = rng.gauss() * 0.1;
      x[static_cast<size_t>(i)] = rng.gauss();
    }
    tile.set_weights(w);
    tile.forward(x); // warm-up: CUDA context, kernels, scratch

    using clock = std::chrono::steady_clock;
    double checksum_analog = 0.0;
    auto t0 = clock::now();
    if (batched) {
      std::vector<float> X(static_cast<size_t>(reps) * size), Y(X.size());
      for (int r = 0; r < reps; ++r)
        for (int j = 0; j < size; ++j)
          X[static_cast<size_t>(r) * size + j] = static_cast<float>(x[static_cast<size_t>(j)]);
      tile.forward_batch(X.data(), reps, Y.data());
      for (float v : Y) checksum_analog += v;
    } else {
      for (int r = 0; r < reps; ++r)
        for (double v : tile.forward(x)) checksum_analog += v;
    }
    auto t1 = clock::now();
    double checksum_digital = 0.0;
    for (int r = 0; r < reps; ++r)
      for (int i = 0; i < size; ++i) {
        double acc = 0.0;
        for (int j = 0; j < size; ++j) acc += w(i, j) * x[static_cast<size_t>(j)];
        checksum_digital += acc;
      }
    auto t2 = clock::now();
    const double analog_s = std::chrono::duration<double>(t1 - t0).count();
    const double digital_s = std::chrono::duration<double>(t2 - t1).count();

    std::ofstream csv(out_dir + "/matvec_bench.csv");
    if (!csv) throw Error("csv: cannot open '" + out_dir + "/matvec_bench.csv' for writing");
    csv << "# relative, informational only; timings vary between runs\n";
    csv << "# analog_elapsed_s=" << fmt_double(analog_s) << "\n";
    csv << "# digital_elapsed_s=" << fmt_double(digital_s) << "\n";
    csv << "# analog_over_digital=" << fmt_double(digital_s > 0.0 ? analog_s / digital_s : 0.0)
        << "\n";
    csv << "# backend=b200" << (batched ? " batched" : " per-call") << "\n";
    csv << "size,reps,checksum_analog,checksum_digital\n";
    csv << size << "," << reps << "," << fmt_double(checksum_analog) << ","
        << fmt_double(checksum_digital) << "\n";
  } catch (const std::exception &e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
