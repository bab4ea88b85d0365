"""The C++ host layer (include/xbarsim_b200/tile.hpp) on the GPU: the
reference's own unit-test cases re-run through the C++ API."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_cpp_parity_driver():
    exe = os.path.join(HERE, "cpp", "test_tile_b200")
    src = os.path.join(HERE, "cpp", "test_tile_b200.cpp")
    if not os.path.exists(exe) or os.path.getmtime(exe) < os.path.getmtime(src):
        subprocess.run(["sh", os.path.join(HERE, "cpp", "build.sh")], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
