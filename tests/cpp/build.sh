#!/bin/sh
# Builds the C++ drivers (tile API, batched NN host) against the in-tree libxbtile.so.
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
for t in test_tile_b200 test_nn_b200 test_shard_b200; do
  g++ -std=c++20 -O2 -Wall -Wextra -pthread -I"$ROOT/include" "$ROOT/tests/cpp/$t.cpp" \
      -L"$ROOT/paper_2104_02184_b200" -lxbtile \
      -Wl,-rpath,'$ORIGIN/../../paper_2104_02184_b200' -o "$ROOT/tests/cpp/$t"
done
# the per-sample C++ bench (bench.py reports it as "per_sample")
g++ -std=c++20 -O2 -Wall -Wextra -I"$ROOT/include" "$ROOT/tools/per_sample_bench.cpp" \
    -L"$ROOT/paper_2104_02184_b200" -lxbtile \
    -Wl,-rpath,'$ORIGIN/../paper_2104_02184_b200' -o "$ROOT/tools/per_sample_bench"
