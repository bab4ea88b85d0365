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
for mode in ("0", "1"):
    os.environ["XB_TC_PAIR"] = mode
    t = xb.AnalogTile(300, 260, xb.TileSettings(mvm_precision=xb.MVM_TF32), 2)
    t.forward(rng.uniform(-1, 1, (48, 260)).astype(np.float32))
    t.backward(rng.uniform(-1, 1, (48, 300)).astype(np.float32))
os.environ["XB_TC_PAIR"] = "0"
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
