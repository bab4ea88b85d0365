"""Small driver for ncu: the north-star update (4096^2 reram_sb, BL 31, B 256)
and forward, `--iters` times each.  Used as
    python tools/profile_pulse.py && ncu --set full -k regex:pulse_kernel -s 1 -c 1 ...
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2104_02184_b200 as xb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--device", default="reram_sb")
ap.add_argument("--precision", type=int, default=xb.MVM_FP32)
ap.add_argument("--warm", type=int, default=0, help="untimed iterations first")
ap.add_argument("--backward", action="store_true", help="also run backward_dev each iteration")
args = ap.parse_args()

dev = xb.device_preset(args.device)
fwd = xb.default_io()
fwd.bound_management = xb.BM_ITERATIVE
cfg = xb.TileSettings(device=dev, forward_io=fwd, mvm_precision=args.precision)
t = xb.AnalogTile(args.n, args.n, cfg, 1234)
s = torch.cuda.Stream()
t.set_stream(s.cuda_stream)
t.set_weights(np.random.default_rng(7).uniform(-0.1, 0.1, (args.n, args.n)).astype(np.float32))
g = torch.Generator(device="cuda")
g.manual_seed(7)
X = torch.rand(args.batch, args.n, device="cuda", generator=g) * 2 - 1
D = torch.rand(args.batch, args.n, device="cuda", generator=g) * 2 - 1
Y = torch.empty(args.batch, args.n, device="cuda")
with torch.cuda.stream(s):
    for _ in range(args.warm):
        t.forward_dev(X, Y)
        t.update_dev(X, D, 0.01)
t.synchronize()
t.set_timing(True)
G = torch.empty(args.batch, args.n, device="cuda")
with torch.cuda.stream(s):
    for _ in range(args.iters):
        t.forward_dev(X, Y)
        if args.backward:
            t.backward_dev(D, G)
        t.update_dev(X, D, 0.01)
tm = t.read_timing()
print(os.environ.get("XBTILE_LIB", "default"),
      {k: (round(v[0] / max(v[1], 1), 4), v[1]) for k, v in tm.items()})
