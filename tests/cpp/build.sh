#!/bin/sh
# Builds the C++ parity driver against the in-tree libxbtile.so.
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
g++ -std=c++20 -O2 -Wall -Wextra -I"$ROOT/include" "$ROOT/tests/cpp/test_tile_b200.cpp" \
    -L"$ROOT/paper_2104_02184_b200" -lxbtile \
    -Wl,-rpath,'$ORIGIN/../../paper_2104_02184_b200' -o "$ROOT/tests/cpp/test_tile_b200"
