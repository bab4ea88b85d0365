// The reference's own NN tests (proj/tests/test_nn.cpp), unmodified and
// compiled where they lie, with every AnalogTile they build replaced by the
// B200 adapter (integration/b200_tile_adapter.hpp): the reference NN host
// (proj/src/nn.cpp: AnalogDenseLayer, AnalogConv2DLayer, Network, train)
// drives the GPU tile through xbarsim::TileBase.  Built by
// integration/Makefile into integration/_ref/ (it needs /root/reference);
// run by tests/test_gpu_cpp.py.
#include "helpers.hpp"          // proj/tests/helpers.hpp (includes xbarsim/tile.hpp)
#include "xbarsim/nn.hpp"
#include "b200_tile_adapter.hpp"

// from here on the test file's AnalogTile is the B200 tile
#define AnalogTile B200AnalogTile
#include "test_nn.cpp"
