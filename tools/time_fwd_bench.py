"""Device time of the bench's forward (4096^2 reram_sb tile after 23 update
steps, batch 256, TF32, default converters) under variants of the output
stage / bound management, each the mean of --iters back-to-back calls
between CUDA events.  An A/B tool, never a bench number:
    python tools/time_fwd_bench.py [--iters 50]"""
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
ap.add_argument("--only", default=None, help="run one variant (perfect, default, noise-off, "
                "bm-iter0, bm); e.g. under ncu")
a = ap.parse_args()
s = torch.cuda.Stream()
torch.cuda.set_stream(s)


def io_of(name):
    io = xb.perfect_io() if name == "perfect" else xb.default_io()
    if name.startswith("bm"):
        io.bound_management = xb.BM_ITERATIVE
    if name == "bm-iter0":
        io.bm_max_iter = 0
    if name == "noise-off":
        io.sigma_out = 0.0
    return io


g = torch.Generator(device="cuda")
g.manual_seed(3)
X = torch.rand(a.batch, a.n, device="cuda", generator=g) * 2 - 1
Y = torch.empty(a.batch, a.n, device="cuda")
base = xb.AnalogTile(a.n, a.n, xb.TileSettings(device=xb.device_preset("reram_sb"),
                                               mvm_precision=xb.MVM_TF32), 5)
base.set_stream(s.cuda_stream)
base.set_weights(np.random.default_rng(7).uniform(-0.1, 0.1, (a.n, a.n)).astype(np.float32))
for _ in range(23):
    base.update_dev(X, torch.rand(a.batch, a.n, device="cuda", generator=g) * 2 - 1, 0.01)
W = base.get_weights()
for name, env in (("perfect", {}), ("default", {}), ("noise-off", {}), ("bm-iter0", {}),
                  ("bm", {}), ("bm", {"XB_BM_NO_LEVEL1": "1"}), ("bm", {"XB_BM_HOST_PASSES": "1"})):
    if a.only and (name != a.only or env):
        continue
    for k in ("XB_BM_NO_LEVEL1", "XB_BM_HOST_PASSES"):
        os.environ.pop(k, None)
    os.environ.update(env)
    io = io_of(name)
    cfg = xb.TileSettings(device=xb.device_preset("reram_sb"), forward_io=io, backward_io=io,
                          mvm_precision=xb.MVM_TF32)
    t = xb.AnalogTile(a.n, a.n, cfg, 5)
    t.set_stream(s.cuda_stream)
    t.set_weights(W)
    for _ in range(3):
        t.forward_dev(X, Y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(a.iters):
        t.forward_dev(X, Y)
    e1.record(s)
    torch.cuda.synchronize()
    print(f"{name:10s} {str(env):32s} {e0.elapsed_time(e1) / a.iters * 1e3:7.2f} us")
