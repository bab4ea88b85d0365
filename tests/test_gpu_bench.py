"""bench.py contract checks on the GPU: the N = 1 line and the N > 1 code
path (the cfg5 16384^2 tile row-sharded over the ranks, max-over-ranks
timing, weak-scaling and inference extras) run as two torchrun ranks.  With
one GPU both ranks share cuda:0, where NCCL cannot join them, so each rank
gets a one-rank communicator (XB_BENCH_DEVICE): this validates the multi-rank
control flow only -- its timings are not measurements and its reductions are
rank-local (the sharded arithmetic itself: tests/test_gpu_comm.py)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline",
        "clocks", "gpu_launches", "e2e"}


def _last_json(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


@pytest.mark.gpu
def test_bench_single_gpu_line():
    r = subprocess.run([sys.executable, "bench.py", "--steps", "2", "--warmup", "3",
                        "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["frac"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0


@pytest.mark.gpu
def test_bench_two_rank_code_path():
    env = dict(os.environ, XB_BENCH_DEVICE="0")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        "29531", "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _last_json(r.stdout)
    assert KEYS <= set(d)
    assert d["n_gpus"] == 2 and d["config"]["tile_rows_total"] == 16384
    assert d["scaling"] == "strong" and d["config"]["rows_per_gpu"] == 8192
    assert d["e2e"]["h2d_bytes_per_step"] == 2 * (256 * 16384 * 4 * 2 + 256 * 8192 * 4)
    assert d["weak_scaling"]["rows_per_gpu"] == 4096 and d["weak_scaling"]["value"] > 0
    assert d["inference_pass"]["drift_to_s"] > 0


@pytest.mark.gpu
def test_launch_floor_measurement():
    """xb_launch_floor_us (the latency floor of cfg1/cfg2's rooflines): empty
    kernels back to back from C cost a few microseconds each on the device."""
    import paper_2104_02184_b200 as xb
    us = xb.launch_floor_us(32, 3)
    assert 0.3 < us < 50.0, us
    with pytest.raises(xb.Error, match="launch_floor"):
        xb.launch_floor_us(0, 1)
