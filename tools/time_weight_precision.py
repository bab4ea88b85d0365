"""Time the 4096^2 reram_sb update (B 256) with fp32 and compensated weights."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2104_02184_b200 as xb  # noqa: E402
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
for wp in (xb.W_FP32, xb.W_FP32X2):
    t = xb.AnalogTile(4096, 4096, xb.TileSettings(device=xb.device_preset("reram_sb"), weight_precision=wp), 3)
    t.set_stream(s.cuda_stream)
    t.set_weights(np.random.default_rng(7).uniform(-0.1, 0.1, (4096, 4096)).astype(np.float32))
    g = torch.Generator(device="cuda"); g.manual_seed(1)
    X = torch.rand(256, 4096, device="cuda", generator=g) * 2 - 1
    D = torch.rand(256, 4096, device="cuda", generator=g) * 2 - 1
    for _ in range(2): t.update_dev(X, D, 0.01)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(5): t.update_dev(X, D, 0.01)
    e1.record(s); torch.cuda.synchronize()
    print(wp, e0.elapsed_time(e1) / 5, "ms")
