"""The C++ host layer (include/xbarsim_b200/tile.hpp, nn.hpp) on the GPU: the
reference's own unit-test cases re-run through the C++ API."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("driver", ["test_tile_b200", "test_nn_b200"])
def test_cpp_parity_driver(driver):
    exe = os.path.join(HERE, "cpp", driver)
    src = os.path.join(HERE, "cpp", driver + ".cpp")
    if not os.path.exists(exe) or os.path.getmtime(exe) < os.path.getmtime(src):
        subprocess.run(["sh", os.path.join(HERE, "cpp", "build.sh")], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
