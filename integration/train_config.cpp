// integration/train_config.cpp -- one config-driven training run, the flow
// of the reference CLI's `train` command (proj/tools/xbarsim_main.cpp:57-80:
// load the config, build dataset and network, check their shapes, train,
// one history row per epoch), on the reference's own config and NN host.
//
// Built twice by integration/Makefile: linked with config.cpp compiled
// plainly (train_config_ref: the reference's CPU tiles) and with the B200
// backend force-included (train_config_b200: every tile build_tile makes is
// a B200 tile, see b200_backend.hpp).  Prints the history as CSV
// (epoch,loss,accuracy) on stdout; tests/test_gpu_cpp.py compares the two.
//
//   train_config_{ref,b200} <config.json> [epochs]
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>

#include "xbarsim/config.hpp"
#include "xbarsim/nn.hpp"

int main(int argc, char **argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s <config.json> [epochs]\n", argv[0]);
    return 2;
  }
  try {
    std::ifstream in(argv[1]);
    if (!in) throw std::runtime_error(std::string("cannot read ") + argv[1]);
    std::stringstream text;
    text << in.rdbuf();
    xbarsim::ExperimentConfig cfg = xbarsim::parse_config(text.str());
    if (argc > 2) cfg.epochs = std::atoi(argv[2]);
    xbarsim::Dataset data = xbarsim::build_dataset(cfg);
    xbarsim::Network net = xbarsim::build_network(cfg);
    if (net.in_size() != data.n_features || net.out_size() != data.n_outputs)
      throw std::runtime_error("network and dataset shapes differ");
    const auto history = xbarsim::train(net, data, xbarsim::build_train_config(cfg));
    std::printf("epoch,loss,accuracy\n");
    for (const auto &e : history) std::printf("%d,%.17g,%.17g\n", e.epoch, e.loss, e.accuracy);
  } catch (const std::exception &e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
