"""PCM program + drift_to on the cfg5 tile (16384^2 reram_sb), device time of
drift_to as the mean of --iters calls between CUDA events (a profiling
driver for tools/profile_round.sh; the bench's number is cfg5's)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2104_02184_b200 as xb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--iters", type=int, default=5)
a = ap.parse_args()
t = xb.AnalogTile(a.n, a.n, xb.TileSettings(device=xb.device_preset("reram_sb")), 5)
target = np.random.default_rng(1).uniform(-0.5, 0.5, (a.n, a.n)).astype(np.float32)
m = xb.InferenceNoiseModel()
t.program(target, m, 11)
s = torch.cuda.ExternalStream(t.stream())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t.drift_to(10.0 * m.t0)
torch.cuda.synchronize()
e0.record(s)
for k in range(a.iters):
    t.drift_to(100.0 * (k + 1) * m.t0)
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
print(f"drift_to {a.n}^2: {ms:.3f} ms, {20.0 * a.n * a.n / (ms * 1e-3) / 1e9:.0f} GB/s")
