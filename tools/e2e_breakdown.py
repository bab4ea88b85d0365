"""Where the end-to-end (host-buffer API) step time goes on the NS workload:
pinned H2D/D2H bandwidth, and the wall time of AnalogTile.forward/update with
host arrays next to the device-resident forward_dev/update_dev.

    python tools/e2e_breakdown.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2104_02184_b200 as xb  # noqa: E402

N, B, LR = 4096, 256, 0.01
fwd = xb.default_io()
fwd.bound_management, fwd.bm_max_iter = xb.BM_ITERATIVE, 10
t = xb.AnalogTile(N, N, xb.TileSettings(device=xb.device_preset("reram_sb"), forward_io=fwd,
                                        mvm_precision=xb.MVM_TF32), 3)  # the bench's tile
t.set_weights(np.random.default_rng(7).uniform(-0.1, 0.1, (N, N)).astype(np.float32))
g = torch.Generator().manual_seed(1)
X = (torch.rand(B, N, generator=g) * 2 - 1).pin_memory()
D = (torch.rand(B, N, generator=g) * 2 - 1).pin_memory()
Y = torch.empty(B, N).pin_memory()
Xn, Dn, Yn = X.numpy(), D.numpy(), Y.numpy()
dX, dD, dY = X.cuda(), D.cuda(), torch.empty(B, N, device="cuda")


def wall(fn, n=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


s = torch.cuda.current_stream()
print(f"H2D 4 MiB pinned: {wall(lambda: dX.copy_(X, non_blocking=True)):.3f} ms")
print(f"D2H 4 MiB pinned: {wall(lambda: Y.copy_(dY, non_blocking=True)):.3f} ms")
t.set_stream(s.cuda_stream)
print(f"forward_dev:      {wall(lambda: t.forward_dev(dX, dY)):.3f} ms")
print(f"forward (host):   {wall(lambda: t.forward(Xn, out=Yn)):.3f} ms")
print(f"update_dev:       {wall(lambda: t.update_dev(dX, dD, LR)):.3f} ms")
print(f"update (host):    {wall(lambda: t.update(Xn, Dn, LR)):.3f} ms")


def step_host():
    t.forward(Xn, out=Yn)
    t.update(Xn, Dn, LR)


def step_dev():
    t.forward_dev(dX, dY)
    t.update_dev(dX, dD, LR)


print(f"step (host API):  {wall(step_host, 20):.3f} ms")
print(f"step (device):    {wall(step_dev, 20):.3f} ms")
