"""CPU checks of the C++ host layer: the header compiles stand-alone with
-Wall -Wextra -Werror and the parity driver links against libxbtile.so."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("g++") is None, reason="no g++")
def test_header_compiles_cleanly(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text('#include "xbarsim_b200/tile.hpp"\n#include "xbarsim_b200/nn.hpp"\n'
                   "int main() { xbarsim_b200::TileSettings s; (void)s;\n"
                   "  xbarsim_b200::Network n; (void)n; return 0; }\n")
    subprocess.run(["g++", "-std=c++20", "-Wall", "-Wextra", "-Werror", "-fsyntax-only",
                    "-I", os.path.join(ROOT, "include"), str(src)], check=True)


@pytest.mark.skipif(shutil.which("g++") is None, reason="no g++")
def test_parity_driver_links():
    subprocess.run(["sh", os.path.join(ROOT, "tests", "cpp", "build.sh")], check=True)
    assert os.path.exists(os.path.join(ROOT, "tests", "cpp", "test_tile_b200"))
    assert os.path.exists(os.path.join(ROOT, "tests", "cpp", "test_nn_b200"))


REF_INCLUDE = "/root/reference/proj/include"


@pytest.mark.skipif(shutil.which("g++") is None or not os.path.isdir(REF_INCLUDE),
                    reason="needs g++ and the reference headers")
def test_adapters_compile_against_the_reference_tilebase(tmp_path):
    """integration/b200_tile_adapter.hpp (B200AnalogTile, B200TransferTile,
    B200UnitCellTile) implements the reference's own xbarsim::TileBase: the
    three build_tile returns type-check against the reference headers."""
    src = tmp_path / "t.cpp"
    src.write_text(
        '#include "b200_tile_adapter.hpp"\n'
        "std::unique_ptr<xbarsim::TileBase> a(const xbarsim::TileSettings &s) {\n"
        "  return std::make_unique<xbarsim::B200AnalogTile>(4, 3, s, 1); }\n"
        "std::unique_ptr<xbarsim::TileBase> b(const xbarsim::TransferSettings &s) {\n"
        "  return std::make_unique<xbarsim::B200TransferTile>(4, 3, s, 1); }\n"
        "std::unique_ptr<xbarsim::TileBase> c(const xbarsim::UnitCellSettings &s) {\n"
        "  return std::make_unique<xbarsim::B200UnitCellTile>(4, 3, s, 1); }\n")
    subprocess.run(["g++", "-std=c++20", "-Wall", "-Wextra", "-fsyntax-only",
                    "-I", os.path.join(ROOT, "integration"), "-I", REF_INCLUDE,
                    "-I", os.path.join(ROOT, "include"), str(src)], check=True)
