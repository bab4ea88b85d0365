"""Small workload touching every kernel of libxbtile.so, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck python tools/sanitize_driver.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_02184_b200 as xb  # noqa: E402

rng = np.random.default_rng(0)
R, C, B = 200, 136, 40
X = rng.uniform(-1, 1, (B, C)).astype(np.float32)
D = rng.uniform(-1, 1, (B, R)).astype(np.float32)
W = rng.uniform(-0.3, 0.3, (R, C)).astype(np.float32)
for name in ("ideal", "reram_sb", "reram_es"):
    for prec in (xb.MVM_FP32, xb.MVM_TF32, xb.MVM_TF32X3):
        io = xb.default_io()
        io.bound_management = xb.BM_ITERATIVE
        s = xb.TileSettings(device=xb.device_preset(name), forward_io=io, backward_io=io,
                            mvm_precision=prec)
        s.temporal.decay_rate, s.temporal.diffusion_sigma = 0.01, 0.001
        t = xb.AnalogTile(R, C, s, 7)
        t.set_weights(W)
        t.forward(X)
        t.backward(D)
        t.update(X, D, 0.05)
        t.end_minibatch()
        t.forward_noisy(X, 0.02)
        c = t.clone()
        c.update(X[:3], D[:3], 0.05)
        m = xb.InferenceNoiseModel()
        t.program(W, m, 3)
        t.drift_to(1e3)
        print(name, prec, "ok", flush=True)
det = xb.TileSettings(device=xb.device_preset("reram_sb"))
det.update.pulse_type = xb.PULSE_DETERMINISTIC
td = xb.AnalogTile(R, C, det, 1)
td.update(X, D, 0.05)
# tcgen05 at odd sizes; the in-kernel bound-management loop (prestaged m = 1
# slab) and the host-driven re-issue passes on a workload that saturates
t = xb.AnalogTile(300, 260, xb.TileSettings(mvm_precision=xb.MVM_TF32), 2)
t.forward(rng.uniform(-1, 1, (48, 260)).astype(np.float32))
t.backward(rng.uniform(-1, 1, (48, 300)).astype(np.float32))
bio = xb.default_io()
bio.bound_management = xb.BM_ITERATIVE
dev = xb.default_device()
dev.w_max, dev.w_min = 1.0, -1.0
Wb = rng.uniform(-0.9, 0.9, (256, 512)).astype(np.float32)
Xb = rng.uniform(-1, 1, (300, 512)).astype(np.float32)
for host in ("0", "1"):
    os.environ["XB_BM_HOST_PASSES"] = host
    for prec in (xb.MVM_TF32, xb.MVM_TF32X3):
        t = xb.AnalogTile(256, 512, xb.TileSettings(device=dev, forward_io=bio, backward_io=bio,
                                                    mvm_precision=prec), 4)
        t.set_weights(Wb)
        t.forward(Xb)
os.environ["XB_BM_HOST_PASSES"] = "0"
# per-sample paths: fused B <= 2, GEMV B <= 15 (forward and backward)
for prec in (xb.MVM_FP32, xb.MVM_TF32X3):
    t = xb.AnalogTile(R, C, xb.TileSettings(device=xb.device_preset("reram_sb"),
                                            mvm_precision=prec), 8)
    t.set_weights(W)
    for b in (1, 2, 5):
        t.forward(X[:b])
        t.backward(D[:b])
        t.update(X[:b], D[:b], 0.05)
# row shards: split-phase backward
import torch  # noqa: E402
sh = [xb.AnalogTile(R, C, xb.TileSettings(), 9, shard=(0, 96)),
      xb.AnalogTile(R, C, xb.TileSettings(), 9, shard=(96, R))]
Dt = torch.from_numpy(D).cuda()
amax = torch.maximum(sh[0].rows_amax(Dt[:, :96].contiguous()), sh[1].rows_amax(Dt[:, 96:].contiguous()))
P = [s_.backward_partial_dev(Dt[:, a:b].contiguous(), amax) for s_, (a, b) in zip(sh, ((0, 96), (96, R)))]
torch.cuda.synchronize()
G = torch.empty(B, C, device="cuda")
sh[0].backward_finish_dev(P[0] + P[1], amax, G)
torch.cuda.synchronize()
tr = xb.TransferSettings()
tr.fast_device = xb.device_preset("reram_sb")
tr.slow_device = xb.device_preset("reram_sb")
tt = xb.TransferTile(R, C, tr, 5)
tt.update(X, D, 0.05)
tt.end_minibatch()
tt.forward(X)
for policy in (xb.UC_ROUND_ROBIN, xb.UC_ALL_TOGETHER):
    u = xb.UnitCellTile(R, C, xb.UnitCellSettings([xb.device_preset("reram_sb")] * 2,
                                                  [1.0, -0.5], policy), 6)
    u.set_weights(W)
    u.update(X, D, 0.05)
    u.forward(X)
    u.backward(D)
print("driver done", flush=True)
