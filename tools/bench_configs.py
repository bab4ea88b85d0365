"""Measure every BASELINE.json config on the B200 path (and the reference on
one host core for a bounded sample).  One JSON line per config.

    python tools/bench_configs.py [--configs 1,2,3,4,5] [--no-ref]

cfg1  256x128 ConstantStep, BL 31, batch 10: forward + backward + update
cfg2  3-layer analog MLP 784-256-128-10 (reram_sb), batch 64, full SGD step
      (sigmoid hidden layers, softmax cross-entropy; a minimal host loop over
      the batched tile API -- the reference NN host is out of scope)
cfg3  4096^2 ExpStep (reram_es, d2d + c2c), BL management, batch 256: update
cfg4  1024^2 Tiki-Taka (A/C reram_sb, units_in_mbatch, transfer_every 2), batch 128
cfg5  16384^2 reram_sb, 1 GPU: forward (default IO + BM) + backward + update of
      256, PCM program + drift_to(1e4 s)
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2104_02184_b200 as xb  # noqa: E402


def ev_time(fn, iters, stream):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(iters):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def rand(shape, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.rand(*shape, device="cuda", generator=g) * 2 - 1


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}


def kbar(t, X, D, lr, samples=16):
    """Measured pulses per cell-update on `samples` samples (sum over slots of
    #x lines firing x #d lines firing, from the trains the update would draw)."""
    c = t.clone()
    xw, dw, _ = c.generate_trains(X[:samples].cpu().numpy(), D[:samples].cpu().numpy(), lr)
    del c
    pulses = 0
    for b in range(xw.shape[0]):
        cx = ((xw[b][:, None] >> np.arange(31, dtype=np.uint32)) & 1).sum(axis=0)
        cd = ((dw[b][:, None] >> np.arange(31, dtype=np.uint32)) & 1).sum(axis=0)
        pulses += int((cx.astype(np.int64) * cd.astype(np.int64)).sum())
    return pulses / (xw.shape[0] * xw.shape[1] * dw.shape[1])


def int_roofline(cells_per_s, kb):
    """(2 + 15 kbar) INT ops per cell-update against the ALU pipe."""
    peak = 148 * 64 * peaks().get("sm_max_mhz", 1965.0) * 1e6
    return {"bound": "int-pipe", "kbar": round(kb, 4),
            "frac": (2.0 + 15.0 * kb) * cells_per_s / peak}


def ref_oracle():
    import oracle
    impl = "reference" if oracle.available("reference") else "restatement"
    return oracle.load(impl), impl


def cfg1(args, stream):
    t = xb.AnalogTile(256, 128, xb.TileSettings(), 1)
    t.set_stream(stream.cuda_stream)
    t.set_weights(np.random.default_rng(7).uniform(-0.1, 0.1, (256, 128)))
    X, D = rand((10, 128), 1), rand((10, 256), 2)
    Y, G = torch.empty(10, 256, device="cuda"), torch.empty(10, 128, device="cuda")

    def step():
        t.forward_dev(X, Y)
        t.backward_dev(D, G)
        t.update_dev(X, D, 0.01)
    ms = ev_time(step, 200, stream)
    out = {"config": "cfg1 256x128 ConstantStep BL31 batch10 fwd+bwd+update", "ms_per_step": ms,
           "cell_updates_per_s": 256 * 128 * 10 / (ms * 1e-3)}
    if not args.no_ref:
        O, impl = ref_oracle()
        o = O.tile(256, 128, O.default("tile"), 1)
        o.set_weights(np.random.default_rng(7).uniform(-0.1, 0.1, (256, 128)))
        x, d = X.cpu().numpy().astype(np.float64), D.cpu().numpy().astype(np.float64)
        t0 = time.perf_counter()
        for b in range(10):
            o.forward(x[b])
            o.backward(d[b])
            o.update(x[b], d[b], 0.01)
        el = time.perf_counter() - t0
        out["ref_1core_ms_per_step"] = el * 1e3
        out["speedup_vs_ref_1core"] = el * 1e3 / ms
    return out


def cfg2(args, stream):
    """784-256-128-10 analog MLP, reram_sb, batch 64, one SGD step."""
    sizes = [784, 256, 128, 10]
    B, lr = 64, 0.01
    cfgs = xb.TileSettings(device=xb.device_preset("reram_sb"))
    tiles = []
    for k in range(3):
        t = xb.AnalogTile(sizes[k + 1], sizes[k], cfgs, 100 + k)
        t.set_stream(stream.cuda_stream)
        bound = 1.0 / np.sqrt(sizes[k])
        t.set_weights(np.random.default_rng(k).uniform(-bound, bound, (sizes[k + 1], sizes[k])))
        tiles.append(t)
    g = torch.Generator(device="cuda").manual_seed(5)
    X = torch.rand(B, 784, device="cuda", generator=g)
    labels = torch.randint(0, 10, (B,), device="cuda", generator=g)
    acts = [X] + [torch.empty(B, n, device="cuda") for n in sizes[1:]]

    def step():
        for k, t in enumerate(tiles):           # forward (sigmoid hidden, logits out)
            t.forward_dev(acts[k], acts[k + 1])
            if k < 2:
                acts[k + 1].sigmoid_()
        p = torch.softmax(acts[3], dim=1)
        delta = p
        delta[torch.arange(B, device="cuda"), labels] -= 1.0
        deltas = [None, None, None]
        deltas[2] = delta.contiguous()
        for k in (2, 1):                         # backward through the tiles
            gin = torch.empty(B, sizes[k], device="cuda")
            tiles[k].backward_dev(deltas[k], gin)
            a = acts[k]
            deltas[k - 1] = (gin * a * (1 - a)).contiguous()
        for k in range(3):                       # pulsed updates, d = -grad / B
            tiles[k].update_dev(acts[k], (-deltas[k] / B).contiguous(), lr)
    ms = ev_time(step, 50, stream)
    out = {"config": "cfg2 MLP 784-256-128-10 reram_sb batch64 SGD step", "ms_per_step": ms,
           "steps_per_s": 1e3 / ms}
    if not args.no_ref:
        O, impl = ref_oracle()
        s = O.default("tile")
        s.device = O.preset("reram_sb")
        ot = [O.tile(sizes[k + 1], sizes[k], s, 100 + k) for k in range(3)]
        xs = X.cpu().numpy().astype(np.float64)
        lab = labels.cpu().numpy()
        sig = lambda v: 1.0 / (1.0 + np.exp(-v))  # noqa: E731
        t0 = time.perf_counter()
        for b in range(8):  # bounded sample: 8 of the 64 samples, scaled to 64
            a0 = xs[b]
            a1 = sig(ot[0].forward(a0))
            a2 = sig(ot[1].forward(a1))
            y = ot[2].forward(a2)
            p = np.exp(y - y.max())
            p /= p.sum()
            p[lab[b]] -= 1.0
            g1 = ot[2].backward(p) * a2 * (1 - a2)
            g0 = ot[1].backward(g1) * a1 * (1 - a1)
            ot[2].update(a2, -p / B, lr)
            ot[1].update(a1, -g1 / B, lr)
            ot[0].update(a0, -g0 / B, lr)
        el = (time.perf_counter() - t0) * 64 / 8
        out["ref_1core_ms_per_step"] = el * 1e3
        out["speedup_vs_ref_1core"] = el * 1e3 / ms
    return out


def update_cfg(name, preset, n, B, blm, args, stream, ref_samples=1):
    dev = xb.device_preset(preset)
    c = xb.TileSettings(device=dev)
    c.update.bl_management = blm
    t = xb.AnalogTile(n, n, c, 3)
    t.set_stream(stream.cuda_stream)
    t.set_weights(np.random.default_rng(7).uniform(-0.1, 0.1, (n, n)).astype(np.float32))
    X, D = rand((B, n), 1), rand((B, n), 2)
    ms = ev_time(lambda: t.update_dev(X, D, 0.01), 5, stream)
    out = {"config": name, "ms_per_batch": ms, "cell_updates_per_s": n * n * B / (ms * 1e-3)}
    out["roofline"] = int_roofline(out["cell_updates_per_s"], kbar(t, X, D, 0.01))
    if not args.no_ref:
        O, impl = ref_oracle()
        s = O.default("tile")
        s.device = O.preset(preset)
        s.update.bl_management = blm
        o = O.tile(n, n, s, 3)
        o.set_weights(np.random.default_rng(7).uniform(-0.1, 0.1, (n, n)))
        x, d = X[:ref_samples].cpu().numpy(), D[:ref_samples].cpu().numpy()
        t0 = time.perf_counter()
        for b in range(ref_samples):
            o.update(x[b].astype(np.float64), d[b].astype(np.float64), 0.01)
        el = (time.perf_counter() - t0) / ref_samples
        out["ref_1core_cell_updates_per_s"] = n * n / el
        out["speedup_vs_ref_1core"] = out["cell_updates_per_s"] / out["ref_1core_cell_updates_per_s"]
    return out


def cfg4(args, stream):
    s = xb.TransferSettings()
    s.fast_device = xb.device_preset("reram_sb")
    s.fast_device.dw_min_dtod = 0.1
    s.slow_device = xb.device_preset("reram_sb")
    s.slow_device.dw_min_std = 0.2
    s.units_in_mbatch, s.transfer_every, s.transfer_lr = 1, 2, 0.1
    s.columns_per_event, s.gamma = 1, 1.0
    t = xb.TransferTile(1024, 1024, s, 1234)
    X = np.random.default_rng(1).uniform(-1, 1, (128, 1024)).astype(np.float32)
    D = np.random.default_rng(2).uniform(-1, 1, (128, 1024)).astype(np.float32)

    def batch():
        t.update(X, D, 0.01)
        t.end_minibatch()
    for _ in range(2):
        batch()
    t0 = time.perf_counter()
    n = 10
    for _ in range(n):
        batch()
    ms = (time.perf_counter() - t0) / n * 1e3
    return {"config": "cfg4 1024^2 Tiki-Taka reram_sb units_in_mbatch every2 batch128 (host API)",
            "ms_per_batch": ms, "cell_updates_per_s": 1024 * 1024 * 128 / (ms * 1e-3),
            "transfer_events": t.transfer_events()}


def cfg5(args, stream):
    n, B = 16384, 256
    fwd = xb.default_io()
    fwd.bound_management = xb.BM_ITERATIVE
    c = xb.TileSettings(device=xb.device_preset("reram_sb"), forward_io=fwd,
                        mvm_precision=xb.MVM_TF32)
    t = xb.AnalogTile(n, n, c, 5)
    t.set_stream(stream.cuda_stream)
    t.set_weights(np.random.default_rng(7).uniform(-0.1, 0.1, (n, n)).astype(np.float32))
    X, D = rand((B, n), 1), rand((B, n), 2)
    Y, G = torch.empty(B, n, device="cuda"), torch.empty(B, n, device="cuda")
    f_ms = ev_time(lambda: t.forward_dev(X, Y), 5, stream)
    b_ms = ev_time(lambda: t.backward_dev(D, G), 3, stream)
    u_ms = ev_time(lambda: t.update_dev(X, D, 0.01), 2, stream)
    m = xb.InferenceNoiseModel()
    target = np.random.default_rng(3).uniform(-0.3, 0.3, (n, n)).astype(np.float32)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    t.program(target, m, 11)
    p_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    t.drift_to(1e4)
    d_s = time.perf_counter() - t0
    mvm_bytes = 4.0 * n * n + 4.0 * B * 2 * n  # W once + x and y
    hbm = peaks().get("hbm_gbs", 6650.0)
    return {"config": "cfg5 16384^2 reram_sb 1 GPU", "forward_ms": f_ms,
            "forward_samples_per_s": B / (f_ms * 1e-3), "backward_ms": b_ms, "update_ms": u_ms,
            "update_cell_updates_per_s": n * n * B / (u_ms * 1e-3),
            "roofline_update": int_roofline(n * n * B / (u_ms * 1e-3), kbar(t, X, D, 0.01)),
            "roofline_mvm_hbm_frac": {"forward": mvm_bytes / (f_ms * 1e-3) / 1e9 / hbm,
                                      "backward": mvm_bytes / (b_ms * 1e-3) / 1e9 / hbm},
            "program_s_incl_h2d_of_target": p_s, "drift_to_s": d_s,
            "ref_1core": "SURVEY §6: program 29.5 s, drift_to 10.9 s, update 33.5 s/sample, "
                         "forward 1.10 s/sample"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--no-ref", action="store_true")
    args = ap.parse_args()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    for c in args.configs.split(","):
        if c == "1":
            r = cfg1(args, stream)
        elif c == "2":
            r = cfg2(args, stream)
        elif c == "3":
            r = update_cfg("cfg3 4096^2 reram_es BL31+BLmgmt batch256 update", "reram_es", 4096,
                           256, 1, args, stream)
        elif c == "4":
            r = cfg4(args, stream)
        elif c == "5":
            r = cfg5(args, stream)
        else:
            continue
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
