"""Device time of the noisy forward / backward MVM (TF32 tcgen05), batch 256:
    XBTILE_LIB=... python tools/time_mvm.py [--n 4096] [--iters 50]
default IO (DAC/ADC, noise, bound management) and the perfect IO, each as the
mean over --iters back-to-back calls between CUDA events."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2104_02184_b200 as xb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--iters", type=int, default=50)
ap.add_argument("--precision", type=int, default=xb.MVM_TF32)
a = ap.parse_args()
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
res = {}
for name, io in (("default", xb.default_io()), ("perfect", xb.perfect_io())):
    cfg = xb.TileSettings(device=xb.device_preset("reram_sb"), forward_io=io, backward_io=io,
                          mvm_precision=a.precision)
    t = xb.AnalogTile(a.n, a.n, cfg, 5)
    t.set_stream(s.cuda_stream)
    t.set_weights(np.random.default_rng(7).uniform(-0.1, 0.1, (a.n, a.n)).astype(np.float32))
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    X = torch.rand(a.batch, a.n, device="cuda", generator=g) * 2 - 1
    Y = torch.empty(a.batch, a.n, device="cuda")
    for fn, key in ((lambda: t.forward_dev(X, Y), "fwd"), (lambda: t.backward_dev(X, Y), "bwd")):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(a.iters):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / a.iters * 1e3
        res[f"{name}_{key}_us"] = round(us, 1)
        # algorithmic HBM bytes of one call: W once + inputs + outputs
        res[f"{name}_{key}_hbm_frac"] = round((4.0 * a.n * a.n + 8.0 * a.batch * a.n) /
                                              (us * 1e-6) / 6.5259e12, 3)
print(os.environ.get("XBTILE_LIB", "default").split("/")[-1], a.n, res)
