"""Digest of the weights after NS-shaped updates (bit-identity checks between
library variants) plus the update time:

    XBTILE_LIB=... python tools/update_digest.py [--device reram_sb] [--n 4096]
"""
import argparse
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2104_02184_b200 as xb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--device", default="reram_sb")
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--batch", type=int, default=256)
a = ap.parse_args()
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
t = xb.AnalogTile(a.n, a.n, xb.TileSettings(device=xb.device_preset(a.device)), 3)
t.set_stream(s.cuda_stream)
t.set_weights(np.random.default_rng(7).uniform(-0.1, 0.1, (a.n, a.n)).astype(np.float32))
g = torch.Generator(device="cuda")
g.manual_seed(1)
X = torch.rand(a.batch, a.n, device="cuda", generator=g) * 2 - 1
D = torch.rand(a.batch, a.n, device="cuda", generator=g) * 2 - 1
t.update_dev(X, D, 0.01)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(3):
    t.update_dev(X, D, 0.01)
e1.record(s)
torch.cuda.synchronize()
w = t.get_weights()
print(os.environ.get("XBTILE_LIB", "default").split("/")[-1], a.device,
      hashlib.sha256(w.tobytes()).hexdigest()[:16], f"{e0.elapsed_time(e1) / 3:.3f} ms")
