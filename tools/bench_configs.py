"""Every BASELINE.json config on the B200 path, each with its roofline, the
reference CPU path on one host core (a bounded sample, the -O2 -march=native
build of the reference sources) and an end-to-end number through the public
host-buffer API.  Used by bench.py (`--config cfgN` prints one contract line;
the default NS line embeds a summary of all five under "configs") and runnable
alone:

    python tools/bench_configs.py [--configs 1,2,3,4,5] [--no-ref]

cfg1  256x128 ConstantStep, BL 31, batch 10: forward + backward + update
cfg2  3-layer analog MLP 784-256-128-10 (reram_sb), batch 64, one SGD step
      (sigmoid hidden layers, softmax cross-entropy; the batched tile API
      driven from a minimal host loop -- the reference NN host is out of scope)
cfg3  4096^2 ExpStep (reram_es, d2d + c2c), BL management, batch 256: update
cfg4  1024^2 Tiki-Taka (A/C reram_sb, units_in_mbatch, transfer_every 2), batch 128
cfg5  16384^2 reram_sb, 1 GPU: forward (default IO + BM), backward, update of
      256; PCM program + drift_to(1e4 s)
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

UNIT_CU = "cell-updates/s"


def ev_time(fn, iters, stream, warm=2):
    """Device time (CUDA events on the tile stream) per call, after warm-up."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(iters):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def wall_time(fn, iters, warm=1):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(iters):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / iters * 1e3


def rand(shape, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.rand(*shape, device="cuda", generator=g) * 2 - 1


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


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


def int_roofline(cells_per_s, kb, kernel="pulse_kernel"):
    """(2 + 15 kbar) INT ops per cell-update against the ALU pipe."""
    pk, kind = peaks()
    peak = 148 * 64 * pk.get("sm_max_mhz", 1965.0) * 1e6
    ach = (2.0 + 15.0 * kb) * cells_per_s
    return {"bound": "int-pipe", "achieved": ach / 1e9, "peak": peak / 1e9, "unit": "Gop/s",
            "frac": ach / peak, "kbar": round(kb, 4), "kernel": kernel,
            "basis": "SURVEY 8d: (2 + 15 kbar) INT ops per cell-update",
            "peak_kind": f"148 SM x 64 ALU lanes x sm_max_mhz ({kind})"}


def hbm_roofline(bytes_, ms, what):
    pk, kind = peaks()
    ach = bytes_ / (ms * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": ach / pk["hbm_gbs"], "basis": what, "peak_kind": kind}


def launch_floor_us(stream, iters=200):
    """Device time per launch of empty kernels issued back to back from C
    (xb_launch_floor_us): the per-launch floor a latency-bound step cannot go
    under (a floor measured through Python would include the interpreter)."""
    return xb.launch_floor_us(64, 5)


def latency_roofline(ms, launches, floor_us):
    """Latency-bound steps: floor = launches x the single-launch floor."""
    floor = launches * floor_us * 1e-3
    return {"bound": "launch-latency", "achieved": ms, "peak": floor, "unit": "ms/step",
            "frac": floor / ms, "launches_per_step": launches,
            "basis": f"{launches} dependent launches x {floor_us:.2f} us (measured: empty "
                     "kernels issued back to back from C)"}


def ref_oracle():
    """The reference's own sources (-O2 -march=native build when the CPU runs
    it): the timed CPU arm."""
    import oracle
    for impl in ("reference_native", "reference", "restatement"):
        if oracle.available(impl):
            return oracle.load(impl), impl
    oracle.build(reference=False)
    return oracle.load("restatement"), "restatement"


def cpu_line(value, unit, sample, impl):
    return {"value": value, "unit": unit, "cores": 1,
            "kind": "port" if impl == "restatement" else "reference", "build": impl,
            "sample": sample}


def launches_in(fn):
    n0 = xb.launch_count()
    fn()
    torch.cuda.synchronize()
    return xb.launch_count() - n0


# ------------------------------------------------------------------ cfg1
def cfg1(args, stream):
    R, C, B = 256, 128, 10
    t = xb.AnalogTile(R, C, xb.TileSettings(), 1)
    t.set_stream(stream.cuda_stream)
    W0 = np.random.default_rng(7).uniform(-0.1, 0.1, (R, C)).astype(np.float32)
    t.set_weights(W0)
    X, D = rand((B, C), 1), rand((B, R), 2)
    Y, G = torch.empty(B, R, device="cuda"), torch.empty(B, C, device="cuda")

    def step():
        t.forward_dev(X, Y)
        t.backward_dev(D, G)
        t.update_dev(X, D, 0.01)
    ms = ev_time(step, 200, stream)
    nl = launches_in(step)
    out = {"metric": "cell-updates/s (cfg1 step: forward + backward + update of 10 samples)",
           "value": R * C * B / (ms * 1e-3), "unit": UNIT_CU, "ms_per_step": ms,
           "higher_is_better": True, "gpu_launches": nl,
           "config": {"workload": "cfg1: 256x128 ConstantStep tile, BL 31, batch 10: noisy "
                                  "forward + backward + stochastic pulsed update"},
           "roofline": latency_roofline(ms, nl, launch_floor_us(stream))}
    Xh, Dh = X.cpu().numpy(), D.cpu().numpy()
    e_ms = wall_time(lambda: (t.forward(Xh), t.backward(Dh), t.update(Xh, Dh, 0.01)), 50)
    out["e2e"] = {"value": R * C * B / (e_ms * 1e-3), "unit": UNIT_CU,
                  "h2d_bytes_per_step": 4 * B * (2 * C + 2 * R), "d2h_bytes_per_step": 4 * B * (R + C),
                  "api": "AnalogTile.forward / backward / update with host arrays"}
    if not args.no_ref:
        O, impl = ref_oracle()
        o = O.tile(R, C, O.default("tile"), 1)
        o.set_weights(W0.astype(np.float64))
        x, d = Xh.astype(np.float64), Dh.astype(np.float64)
        t0 = time.perf_counter()
        for _ in range(5):
            for b in range(B):
                o.forward(x[b])
                o.backward(d[b])
                o.update(x[b], d[b], 0.01)
        el = (time.perf_counter() - t0) / 5
        out["cpu_baseline"] = cpu_line(R * C * B / el, UNIT_CU,
                                       "5 steps of 10 (forward, backward, update) samples", impl)
    return out


# ------------------------------------------------------------------ cfg2
def cfg2(args, stream):
    """784-256-128-10 analog MLP, reram_sb, batch 64, one SGD step."""
    sizes = [784, 256, 128, 10]
    B, lr = 64, 0.01
    cfgs = xb.TileSettings(device=xb.device_preset("reram_sb"))
    tiles, Ws = [], []
    for k in range(3):
        t = xb.AnalogTile(sizes[k + 1], sizes[k], cfgs, 100 + k)
        t.set_stream(stream.cuda_stream)
        bound = 1.0 / np.sqrt(sizes[k])
        Ws.append(np.random.default_rng(k).uniform(-bound, bound, (sizes[k + 1], sizes[k]))
                  .astype(np.float32))
        t.set_weights(Ws[-1])
        tiles.append(t)
    g = torch.Generator(device="cuda").manual_seed(5)
    X = torch.rand(B, 784, device="cuda", generator=g)
    labels = torch.randint(0, 10, (B,), device="cuda", generator=g)
    acts = [X] + [torch.empty(B, n, device="cuda") for n in sizes[1:]]
    # the step's glue (activations, loss gradient, scaling) as few torch ops
    # on preallocated buffers: the step is enqueue-bound, not GPU-bound
    onehot = torch.zeros(B, 10, device="cuda")
    onehot[torch.arange(B, device="cuda"), labels] = 1.0
    gins = [None] + [torch.empty(B, sizes[k], device="cuda") for k in (1, 2)]
    deltas = [torch.empty(B, sizes[k + 1], device="cuda") for k in range(3)]
    slope = [None] + [torch.empty(B, sizes[k], device="cuda") for k in (1, 2)]
    upd = [torch.empty(B, sizes[k + 1], device="cuda") for k in range(3)]

    def step():
        for k, t in enumerate(tiles):           # forward (sigmoid hidden, logits out)
            t.forward_dev(acts[k], acts[k + 1])
            if k < 2:
                torch.sigmoid(acts[k + 1], out=acts[k + 1])
        torch.sub(torch.softmax(acts[3], dim=1), onehot, out=deltas[2])  # softmax CE grad
        for k in (2, 1):                         # backward through the tiles
            tiles[k].backward_dev(deltas[k], gins[k])
            torch.addcmul(acts[k], acts[k], acts[k], value=-1.0, out=slope[k])  # a (1 - a)
            torch.mul(gins[k], slope[k], out=deltas[k - 1])
        for k in range(3):                       # pulsed updates, d = -grad / B
            torch.mul(deltas[k], -1.0 / B, out=upd[k])
            tiles[k].update_dev(acts[k], upd[k], lr)
    ms = ev_time(step, 50, stream)
    nl = launches_in(step)
    cells = sum(sizes[k] * sizes[k + 1] for k in range(3)) * B
    out = {"metric": "SGD steps/s (cfg2: 784-256-128-10 analog MLP, batch 64)",
           "value": 1e3 / ms, "unit": "steps/s", "ms_per_step": ms, "higher_is_better": True,
           "gpu_launches": nl, "cell_updates_per_s": cells / (ms * 1e-3),
           "config": {"workload": "cfg2: 3 reram_sb tiles 784-256-128-10, sigmoid hidden "
                                  "layers, softmax cross-entropy, batch 64, synthetic MNIST-"
                                  "shaped data; one SGD step = 64 forwards, 64 backwards, "
                                  "64 pulsed updates per tile (batched calls)"},
           "roofline": latency_roofline(ms, nl, launch_floor_us(stream))}
    # e2e: the step through the host-buffer API (numpy activations)
    Xh, lab = X.cpu().numpy(), labels.cpu().numpy()
    sig = lambda v: 1.0 / (1.0 + np.exp(-v))  # noqa: E731

    def host_step():
        a = [Xh]
        for k in range(3):
            y = tiles[k].forward(a[-1])
            a.append(sig(y).astype(np.float32) if k < 2 else y)
        p = np.exp(a[3] - a[3].max(axis=1, keepdims=True))
        p /= p.sum(axis=1, keepdims=True)
        p[np.arange(B), lab] -= 1.0
        dl = [None, None, p.astype(np.float32)]
        for k in (2, 1):
            gin = tiles[k].backward(dl[k])
            dl[k - 1] = (gin * a[k] * (1 - a[k])).astype(np.float32)
        for k in range(3):
            tiles[k].update(a[k], -dl[k] / B, lr)
    e_ms = wall_time(host_step, 20)
    out["e2e"] = {"value": 1e3 / e_ms, "unit": "steps/s",
                  "h2d_bytes_per_step": 4 * B * (2 * sum(sizes[:3]) + 2 * sum(sizes[1:]) + sizes[1] + sizes[2]),
                  "d2h_bytes_per_step": 4 * B * (sum(sizes[1:]) + sizes[1] + sizes[2]),
                  "api": "AnalogTile.forward / backward / update with host arrays per layer"}
    if not args.no_ref:
        O, impl = ref_oracle()
        s = O.default("tile")
        s.device = O.preset("reram_sb")
        ot = []
        for k in range(3):
            o = O.tile(sizes[k + 1], sizes[k], s, 100 + k)
            o.set_weights(Ws[k].astype(np.float64))
            ot.append(o)
        xs = Xh.astype(np.float64)
        t0 = time.perf_counter()
        n = 8  # bounded sample: 8 of the 64 samples, scaled to the step
        for b in range(n):
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
        el = (time.perf_counter() - t0) * B / n
        out["cpu_baseline"] = cpu_line(1.0 / el, "steps/s",
                                       f"{n} of the 64 samples of a step, scaled to 64", impl)
    return out


# ------------------------------------------------------------------ cfg3
def cfg3(args, stream, ref_samples=1):
    n, B, preset = 4096, 256, "reram_es"
    c = xb.TileSettings(device=xb.device_preset(preset))
    c.update.bl_management = 1
    t = xb.AnalogTile(n, n, c, 3)
    t.set_stream(stream.cuda_stream)
    W0 = np.random.default_rng(7).uniform(-0.1, 0.1, (n, n)).astype(np.float32)
    t.set_weights(W0)
    X, D = rand((B, n), 1), rand((B, n), 2)
    ms = ev_time(lambda: t.update_dev(X, D, 0.01), 5, stream)
    nl = launches_in(lambda: t.update_dev(X, D, 0.01))
    cps = n * n * B / (ms * 1e-3)
    out = {"metric": "cell-updates/s (cfg3: pulsed update, 4096^2 ExpStep, BL management)",
           "value": cps, "unit": UNIT_CU, "ms_per_step": ms, "higher_is_better": True,
           "gpu_launches": nl,
           "config": {"workload": "cfg3: 4096x4096 reram_es (ExpStep, d2d 0.3, c2c 0.3, "
                                  "up_down 0.1), BL 31 with BL management, batch 256, lr 0.01"},
           "roofline": int_roofline(cps, kbar(t, X, D, 0.01), "pulse_kernel<EXP_STEP,noise>")}
    Xh, Dh = X.cpu().numpy(), D.cpu().numpy()
    e_ms = wall_time(lambda: t.update(Xh, Dh, 0.01), 3)
    out["e2e"] = {"value": n * n * B / (e_ms * 1e-3), "unit": UNIT_CU,
                  "h2d_bytes_per_step": 4 * B * 2 * n, "d2h_bytes_per_step": 0,
                  "api": "AnalogTile.update(X host, D host)"}
    if not args.no_ref:
        O, impl = ref_oracle()
        s = O.default("tile")
        s.device = O.preset(preset)
        s.update.bl_management = 1
        o = O.tile(n, n, s, 3)
        o.set_weights(W0.astype(np.float64))
        x, d = Xh[:ref_samples].astype(np.float64), Dh[:ref_samples].astype(np.float64)
        t0 = time.perf_counter()
        for b in range(ref_samples):
            o.update(x[b], d[b], 0.01)
        el = (time.perf_counter() - t0) / ref_samples
        out["cpu_baseline"] = cpu_line(n * n / el, UNIT_CU,
                                       f"{ref_samples} AnalogTile::update sample(s)", impl)
    return out


# ------------------------------------------------------------------ cfg4
def cfg4(args, stream):
    n, B = 1024, 128
    s = xb.TransferSettings()
    s.fast_device = xb.device_preset("reram_sb")
    s.fast_device.dw_min_dtod = 0.1
    s.slow_device = xb.device_preset("reram_sb")
    s.slow_device.dw_min_std = 0.2
    s.units_in_mbatch, s.transfer_every, s.transfer_lr = 1, 2, 0.1
    s.columns_per_event, s.gamma = 1, 1.0
    t = xb.TransferTile(n, n, s, 1234)
    fast = t.fast_tile()
    X, D = rand((B, n), 1), rand((B, n), 2)

    def batch():  # one mini-batch: B updates of A, end_minibatch (a transfer every 2nd)
        fast.update_dev(X, D, 0.01)
        t.end_minibatch()
    fs = torch.cuda.ExternalStream(fast.stream())
    ms = ev_time(batch, 20, fs)
    nl = launches_in(batch) + launches_in(batch)  # two mini-batches: one transfer
    cps = n * n * B / (ms * 1e-3)
    out = {"metric": "cell-updates/s (cfg4: Tiki-Taka mini-batch, 1024^2, batch 128)",
           "value": cps, "unit": UNIT_CU, "ms_per_step": ms, "higher_is_better": True,
           "gpu_launches_per_2_batches": nl,
           "config": {"workload": "cfg4: 1024x1024 Tiki-Taka (A, C reram_sb; A dtod 0.1, C "
                                  "std 0.2), units_in_mbatch, transfer_every 2, transfer_lr "
                                  "0.1, 1 column per event, gamma 1, batch 128"},
           "roofline": int_roofline(cps, kbar(fast, X, D, 0.01))}
    Xh, Dh = X.cpu().numpy(), D.cpu().numpy()

    def host_batch():
        t.update(Xh, Dh, 0.01)
        t.end_minibatch()
    e_ms = wall_time(host_batch, 10)
    out["e2e"] = {"value": n * n * B / (e_ms * 1e-3), "unit": UNIT_CU,
                  "h2d_bytes_per_step": 4 * B * 2 * n, "d2h_bytes_per_step": 0,
                  "api": "TransferTile.update(X, D host) + end_minibatch"}
    if not args.no_ref:
        O, impl = ref_oracle()
        rs = O.default("transfer")
        rs.fast_device = O.preset("reram_sb")
        rs.fast_device.dw_min_dtod = 0.1
        rs.slow_device = O.preset("reram_sb")
        rs.slow_device.dw_min_std = 0.2
        rs.units_in_mbatch, rs.transfer_every, rs.transfer_lr = 1, 2, 0.1
        rs.columns_per_event, rs.gamma = 1, 1.0
        o = O.transfer(n, n, rs, 1234)
        x, d = Xh.astype(np.float64), Dh.astype(np.float64)
        m = 4
        t0 = time.perf_counter()
        for b in range(m):
            o.update(x[b], d[b], 0.01)
        o.end_minibatch()
        o.end_minibatch()  # one transfer event (every 2nd mini-batch)
        el = (time.perf_counter() - t0) / m
        out["cpu_baseline"] = cpu_line(n * n / el, UNIT_CU,
                                       f"{m} TransferTile::update samples + one transfer", impl)
    return out


# ------------------------------------------------------------------ cfg5
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
    u_ms = ev_time(lambda: t.update_dev(X, D, 0.01), 2, stream, warm=1)
    m = xb.InferenceNoiseModel()
    target = np.random.default_rng(3).uniform(-0.3, 0.3, (n, n)).astype(np.float32)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    t.program(target, m, 11)
    p_s = time.perf_counter() - t0
    d_ms = ev_time(lambda: t.drift_to(1e4), 3, stream, warm=1)
    step_ms = f_ms + u_ms
    cps = n * n * B / (step_ms * 1e-3)
    mvm_bytes = 4.0 * n * n + 4.0 * B * 2 * n  # W once + x and y
    out = {"metric": "cell-updates/s (cfg5 step on 1 GPU: noisy forward with BM + pulsed update "
                     "of 256 samples, 16384^2)",
           "value": cps, "unit": UNIT_CU, "ms_per_step": step_ms, "higher_is_better": True,
           "config": {"workload": "cfg5: 16384x16384 reram_sb, 1 GPU (bench.py --gpus N shards "
                                  "it over N), forward default IO + BM (TF32), backward, "
                                  "update BL 31 batch 256, program + drift_to(1e4 s)"},
           "phase_ms": {"forward": f_ms, "backward": b_ms, "update": u_ms,
                        "program_s_incl_h2d_of_target": p_s, "drift_to": d_ms},
           "roofline": int_roofline(n * n * B / (u_ms * 1e-3), kbar(t, X, D, 0.01)),
           "roofline_mvm": {"forward": hbm_roofline(mvm_bytes, f_ms, "4 N^2 + 8 B N bytes"),
                            "backward": hbm_roofline(mvm_bytes, b_ms, "4 N^2 + 8 B N bytes")},
           # drift_to: w0, nu read (8 B) + bounds (8 B) + W written (4 B) per cell
           "roofline_drift": hbm_roofline(20.0 * n * n, d_ms, "20 B per cell")}
    Xh, Dh = X.cpu().numpy(), D.cpu().numpy()
    yh = torch.empty(B, n, dtype=torch.float32).pin_memory().numpy()
    e_ms = wall_time(lambda: (t.forward(Xh, out=yh), t.update(Xh, Dh, 0.01)), 2)
    out["e2e"] = {"value": n * n * B / (e_ms * 1e-3), "unit": UNIT_CU,
                  "h2d_bytes_per_step": 4 * B * 3 * n, "d2h_bytes_per_step": 4 * B * n,
                  "api": "AnalogTile.forward(X host) + update(X, D host)"}
    if not args.no_ref:
        # a 256-row slice of the 16384-column tile: the same per-cell work
        O, impl = ref_oracle()
        s = O.default("tile")
        s.device = O.preset("reram_sb")
        rows = 256
        o = O.tile(rows, n, s, 5)
        o.set_weights(np.random.default_rng(7).uniform(-0.1, 0.1, (rows, n)))
        x, d = X[:2].cpu().numpy().astype(np.float64), D[:2, :rows].cpu().numpy().astype(np.float64)
        t0 = time.perf_counter()
        for b in range(2):
            o.forward(x[b])
            o.update(x[b], d[b], 0.01)
        el = (time.perf_counter() - t0) / 2
        out["cpu_baseline"] = cpu_line(rows * n / el, UNIT_CU,
                                       f"2 forward + update samples on a {rows}x{n} row slice",
                                       impl)
    return out


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5}


def summary(d):
    """The compact per-config record embedded in bench.py's NS line."""
    keep = {"metric": d["metric"], "value": d["value"], "unit": d["unit"],
            "ms_per_step": d["ms_per_step"]}
    if "roofline" in d:
        keep["roofline"] = {k: d["roofline"][k] for k in ("bound", "frac", "achieved", "peak",
                                                          "unit")}
    if "roofline_mvm" in d:
        keep["roofline_mvm_frac"] = {k: v["frac"] for k, v in d["roofline_mvm"].items()}
    if "roofline_drift" in d:
        keep["roofline_drift_frac"] = d["roofline_drift"]["frac"]
    if "cpu_baseline" in d:
        keep["cpu_baseline"] = {k: d["cpu_baseline"][k] for k in ("value", "unit", "cores",
                                                                  "kind", "sample")}
    if "e2e" in d:
        keep["e2e"] = {k: d["e2e"][k] for k in ("value", "unit")}
    return keep


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--no-ref", action="store_true")
    args = ap.parse_args()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    for c in args.configs.split(","):
        fn = CONFIGS.get("cfg" + c.strip())
        if fn:
            print(json.dumps(fn(args, stream)), flush=True)


if __name__ == "__main__":
    main()
