"""The C++ host layer (include/xbarsim_b200/tile.hpp, nn.hpp) on the GPU: the
reference's own unit-test cases re-run through the C++ API."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("driver", ["test_tile_b200", "test_nn_b200", "test_shard_b200"])
def test_cpp_parity_driver(driver):
    exe = os.path.join(HERE, "cpp", driver)
    src = os.path.join(HERE, "cpp", driver + ".cpp")
    if not os.path.exists(exe) or os.path.getmtime(exe) < os.path.getmtime(src):
        subprocess.run(["sh", os.path.join(HERE, "cpp", "build.sh")], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout


def test_matvec_bench_cli(tmp_path, restatement):
    """tools/matvec_bench_b200 = the reference CLI's matvec-bench
    (proj/tools/xbarsim_main.cpp:162-212) on the B200 tile: same workload, same
    CSV.  The digital checksum is the reference's to the last bit (its RNG and
    summation order); the analog one agrees within the default-IO noise."""
    root = os.path.dirname(HERE)
    exe = os.path.join(root, "tools", "matvec_bench_b200")
    src = exe + ".cpp"
    if not os.path.exists(exe) or os.path.getmtime(exe) < os.path.getmtime(src):
        subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(root, "include"), src,
                        "-L", os.path.join(root, "paper_2104_02184_b200"), "-lxbtile",
                        "-Wl,-rpath," + os.path.join(root, "paper_2104_02184_b200"), "-o", exe],
                       check=True)
    size, reps, seed = 48, 3, 1234
    for flag in ([], ["--batched"]):
        out = tmp_path / ("b" if flag else "p")
        subprocess.run([exe, "--size", str(size), "--reps", str(reps), "--seed", str(seed),
                        "--out", str(out), *flag], check=True, timeout=300)
        lines = (out / "matvec_bench.csv").read_text().splitlines()
        body = [ln for ln in lines if not ln.startswith("#")]
        assert body[0] == "size,reps,checksum_analog,checksum_digital"
        s, r, ca, cd = body[1].split(",")
        rng = restatement.rng(seed).derive("bench")
        w = [[0.0] * size for _ in range(size)]
        x = [0.0] * size
        for i in range(size):
            for j in range(size):
                w[i][j] = rng.gauss() * 0.1
            x[i] = rng.gauss()
        want = 0.0
        for _ in range(reps):
            for i in range(size):
                acc = 0.0
                for j in range(size):
                    acc += w[i][j] * x[j]
                want += acc
        assert (s, r) == (str(size), str(reps))
        assert cd == repr(want)
        assert abs(float(ca) - want) < 0.05 * sum(abs(v) for v in x) * reps + 1.0
