// integration/b200_backend.hpp -- the "b200" backend of build_tile
// (proj/src/config.cpp:640-681) as a build-time switch.
//
// Force-included (-include) into the reference's config.cpp, compiled
// unmodified where it lies: the reference headers are pulled in here first
// (include-guarded, so config.cpp's own #includes add nothing), then the
// three tile classes build_tile constructs are bound to their B200 adapters
// for the rest of that translation unit only:
//   single / inference -> xbarsim::B200AnalogTile   (AnalogTile)
//   unit_cell          -> xbarsim::B200UnitCellTile (UnitCellTile)
//   transfer           -> xbarsim::B200TransferTile (TransferTile)
// Every other reference object file (nn.cpp's layers and trainer, the
// dataset generators, compound.cpp) is the reference's own, so a config file
// runs through the reference's parse_config / build_network / train with
// the tiles on the GPU.  (The reference's parse_config rejects unknown keys,
// config.cpp:23-34, so the switch cannot be a new JSON key without editing
// the reference; a maintainer who edits it adds `"backend": "b200"` and the
// three returns of INTEGRATION.md section 5.)
#pragma once

#include "xbarsim/compound.hpp"
#include "xbarsim/config.hpp"
#include "xbarsim/nn.hpp"
#include "xbarsim/tile.hpp"

#include "b200_tile_adapter.hpp"

#define AnalogTile B200AnalogTile
#define UnitCellTile B200UnitCellTile
#define TransferTile B200TransferTile
