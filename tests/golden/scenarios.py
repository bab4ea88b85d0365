"""Deterministic oracle scenarios used to pin the restatement.

Each scenario takes a loaded ``oracle.Oracle`` (either implementation) and
returns a dict of numpy arrays.  ``make_golden.py`` runs them through the
REFERENCE build (``oracle/_ref``) and stores the arrays in
``tests/golden/golden.npz``; ``tests/test_oracle_pin.py`` runs them through
the restatement and requires bit-identical arrays.  The scenarios follow the
reference's own test cases (cited per scenario) at small sizes.
"""
from __future__ import annotations

import ctypes as C

import numpy as np


def _u(seed, shape, scale=1.0):
    return np.random.default_rng(seed).uniform(-scale, scale, shape)


def rng_streams(O):
    """proj/src/rng.cpp:14-71 -- derivation, u64, uniform, gauss, bernoulli."""
    out = {}
    r = O.rng(1234)
    out["u64"] = np.array([r.next_u64() for _ in range(700)], dtype=np.uint64)  # > 312: regen
    out["uniform"] = np.array([r.uniform() for _ in range(50)])
    out["gauss"] = np.array([r.gauss() for _ in range(51)])  # odd count exercises the spare
    out["bern"] = np.array([r.bernoulli(p) for p in np.linspace(-0.1, 1.1, 40)], dtype=np.int8)
    seeds = []
    for name in ("forward", "backward", "update", "temporal", "realize", "temporal_init",
                 "fast", "slow", "tile"):
        seeds.append(r.derive(name).base_seed())
    seeds.append(r.derive("cell_member", 3).base_seed())
    seeds.append(r.derive("program", 0).base_seed())
    out["derived"] = np.array(seeds, dtype=np.uint64)
    return out


def quantizer(O):
    """proj/src/io.cpp:42-56; proj/tests/test_tile.cpp:18-51,406-421."""
    vals = np.concatenate([_u(3, 400, 3.0), [0.0, -0.0, 1.0, -1.0, 0.5, 1e-12, 12.0, -13.0]])
    res = []
    for bits in (0, 1, 2, 4, 7, 9):
        for bound in (0.5, 1.0, 12.0):
            res.append([O.quantize(v, bound, bits) for v in vals])
    return {"q": np.array(res)}


def matvec(O):
    """proj/src/io.cpp:93-149 in every mode (test_tile.cpp:53-266)."""
    out = {}
    w = _u(5, (7, 11), 0.4)
    x = _u(6, 11, 0.9)
    d = _u(7, 7, 0.9)
    r = O.rng(99)
    io = O.default("io")
    out["default_fwd"] = O.analog_matvec(w, x, io, r)
    out["default_bwd"] = O.analog_matvec(w, d, io, r, transposed=True)
    io_all = O.default("io")
    io_all.sigma_inp, io_all.sigma_w, io_all.sigma_out = 0.03, 0.02, 0.05
    out["all_noise_fwd"] = O.analog_matvec(w, x, io_all, r)
    out["all_noise_bwd"] = O.analog_matvec(w, d, io_all, r, transposed=True)
    out["zero_in"] = O.analog_matvec(w, np.zeros(11), io, r)
    pio = O.default("perfect_io")
    out["perfect_fwd"] = O.analog_matvec(w, x, pio, r)
    out["perfect_bwd"] = O.analog_matvec(w, d, pio, r, transposed=True)
    nm = O.default("io")
    nm.noise_management = 0
    nm.sigma_out = 0.0
    out["nm_none"] = O.analog_matvec(w, 3.0 * x, nm, r)
    return out


def devices(O):
    """proj/src/device.cpp:26-77 for all presets and laws."""
    out = {}
    for name in ("ideal", "reram_sb", "reram_es"):
        p = O.preset(name)
        r = O.rng(11)
        cells = []
        for _ in range(20):
            cell = np.zeros(6)
            O.lib.or_realize_cell(p, r.h, cell.ctypes.data_as(C.POINTER(C.c_double)))
            cells.append(cell)
        out[f"cells_{name}"] = np.array(cells)
    for kind in range(4):
        for std in (0.0, 0.3):
            p = O.default("device")
            p.kind, p.dw_min, p.dw_min_dtod, p.dw_min_std = kind, 0.01, 0.3, std
            p.w_max, p.w_min, p.up_down, p.w_max_dtod, p.w_min_dtod = 0.5, -0.4, 0.1, 0.2, 0.2
            p.slope, p.gamma = 0.8, 3.0
            r = O.rng(100 + kind)
            cell = np.zeros(6)
            O.lib.or_realize_cell(p, r.h, cell.ctypes.data_as(C.POINTER(C.c_double)))
            w, trace = 0.0, []
            for t in range(300):
                up = (t // 37) % 2 == 0
                w = O.lib.or_apply_pulse(cell.ctypes.data_as(C.POINTER(C.c_double)), w, int(up),
                                         kind, std, r.h)
                trace.append(w)
            out[f"trace_{kind}_{std}"] = np.array(trace)
    return out


def translate_trains(O):
    """proj/src/pulsed.cpp:25-88 (test_pulsed.cpp:17-108,301-317)."""
    out = {}
    x = _u(21, 13)
    d = _u(22, 9)
    x[3] = 0.0
    for k, (lr, blm, bl) in enumerate([(0.01, 0, 31), (0.01, 1, 31), (0.0001, 1, 31),
                                       (5.0, 0, 31), (0.02, 1, 7)]):
        up = O.default("update")
        up.bl, up.bl_management = bl, blm
        b, px, pd, sx, sd = O.translate(x, d, lr, 0.001, up)
        out[f"bl_{k}"] = np.array([b])
        out[f"px_{k}"], out[f"pd_{k}"] = px, pd
        out[f"sx_{k}"], out[f"sd_{k}"] = sx, sd
        xb, db = O.generate_trains(b, px, pd, O.rng(30 + k))
        out[f"xb_{k}"], out[f"db_{k}"] = xb, db
    return out


def _tile_run(O, settings, d_out, d_in, seed, steps, lr=0.01, with_fb=True):
    t = O.tile(d_out, d_in, settings, seed)
    rng = np.random.default_rng(seed)
    t.set_weights(rng.uniform(-0.1, 0.1, (d_out, d_in)))
    res = []
    for _ in range(steps):
        x = rng.uniform(-1, 1, d_in)
        d = rng.uniform(-1, 1, d_out)
        if with_fb:
            res.append(t.forward(x))
            res.append(t.backward(d))
        t.update(x, d, lr)
    res.append(t.get_weights().ravel())
    return np.concatenate(res)


def tile_updates(O):
    """proj/src/tile.cpp:41-171 + pulsed_update per law (test_pulsed.cpp)."""
    out = {}
    for kind in range(4):
        for noisy in (0, 1):
            s = O.default("tile")
            s.device.kind = kind
            s.device.dw_min = 0.002
            s.device.w_max, s.device.w_min = 0.6, -0.6
            if noisy:
                s.device.dw_min_dtod, s.device.dw_min_std, s.device.up_down_dtod = 0.3, 0.3, 0.01
                s.device.up_down = 0.05
                s.device.w_max_dtod = s.device.w_min_dtod = 0.1
            s.update.bl_management = noisy
            out[f"law{kind}_noise{noisy}"] = _tile_run(O, s, 6, 10, 40 + kind, 4)
    s = O.default("tile")
    s.device = O.preset("reram_es")
    s.update.pulse_type = 1  # deterministic_implicit
    out["deterministic_es"] = _tile_run(O, s, 5, 8, 77, 3, lr=0.05)
    s = O.default("tile")
    s.device = O.preset("reram_sb")
    s.forward_io = O.default("perfect_io")
    s.backward_io = O.default("perfect_io")
    out["perfect_sb"] = _tile_run(O, s, 4, 9, 78, 3)
    # noop updates (test_pulsed.cpp:177-189)
    t = O.tile(3, 3, O.default("tile"), 5)
    t.set_weights(_u(8, (3, 3), 0.3))
    t.update(np.ones(3), np.ones(3), 0.0)
    t.update(np.zeros(3), np.ones(3), 0.1)
    t.update(np.ones(3), np.zeros(3), 0.1)
    out["noop"] = t.get_weights()
    return out


def trains_apply(O):
    """AnalogTile::apply_pulse_trains with flip (proj/src/tile.cpp:158-169)."""
    out = {}
    for kind in range(4):
        s = O.default("tile")
        s.device.kind = kind
        s.device.dw_min = 0.003
        s.device.dw_min_dtod = 0.2
        s.device.dw_min_std = 0.0
        t = O.tile(5, 7, s, 300 + kind)
        t.set_weights(_u(9, (5, 7), 0.2))
        rng = np.random.default_rng(kind)
        xb = (rng.random((11, 7)) < 0.4).astype(np.uint8)
        db = (rng.random((11, 5)) < 0.5).astype(np.uint8)
        sx = rng.choice([-1, 0, 1], 7)
        sd = rng.choice([-1, 1], 5)
        t.apply_pulse_trains(11, xb, db, sx, sd, flip=False)
        t.apply_pulse_trains(11, db[:, :5].repeat(2, axis=1)[:, :7], db, sx, sd, flip=True)
        out[f"apply_{kind}"] = t.get_weights()
    return out


def temporal(O):
    """proj/src/tile.cpp:128-156."""
    s = O.default("tile")
    t = O.tile(6, 6, s, 61)
    t.set_weights(_u(10, (6, 6), 0.5))
    tp = O.default("temporal")
    tp.decay_rate, tp.decay_dtod = 0.1, 0.5
    tp.diffusion_sigma, tp.diffusion_dtod = 0.01, 0.2
    tp.reset_prob, tp.reset_dtod = 0.2, 0.3
    t.apply_temporal_step(tp)
    t.apply_temporal_step(tp)
    return {"temporal": t.get_weights()}


def transfer(O):
    """TransferTile (proj/src/compound.cpp:176-293), tiki_taka.json style."""
    s = O.default("transfer")
    s.fast_device = O.preset("reram_sb")
    s.fast_device.dw_min_dtod = 0.1
    s.slow_device = O.preset("reram_sb")
    s.slow_device.dw_min_std = 0.2
    s.units_in_mbatch, s.transfer_every, s.transfer_lr = 1, 2, 0.1
    s.columns_per_event, s.gamma = 1, 1.0
    t = O.transfer(6, 5, s, 1234)
    rng = np.random.default_rng(3)
    t.set_weights(rng.uniform(-0.1, 0.1, (6, 5)))
    res = []
    for mb in range(5):
        for _ in range(4):
            x = rng.uniform(-1, 1, 5)
            d = rng.uniform(-1, 1, 6)
            res.append(t.forward(x))
            res.append(t.backward(d))
            t.update(x, d, 0.1)
        t.end_minibatch()
    res.append(t.get_weights().ravel())
    res.append(t.fast.get_weights().ravel())
    res.append(t.slow.get_weights().ravel())
    return {"transfer": np.concatenate(res), "events": np.array([t.events()])}


def unitcell(O):
    """UnitCellTile (proj/src/compound.cpp:12-174): a +1/-0.5 reram_sb pair with
    c2c noise under both policies, a zero-gain member in round-robin, and the
    single-device reduction to a plain tile."""
    out = {}
    rng = np.random.default_rng(9)
    for name, policy, gains in (("rr", 0, (1.0, -0.5, 0.0)), ("all", 1, (1.0, -0.5, 0.25))):
        s = O.default("unitcell")
        s.n_devices, s.policy = 3, policy
        for k, g in enumerate(gains):
            s.devices[k] = O.preset("reram_sb")
            s.gains[k] = g
        s.devices[2] = O.preset("reram_es")
        u = O.unitcell(6, 5, s, 4321)
        u.set_weights(rng.uniform(-0.2, 0.2, (6, 5)))
        res = []
        for step in range(8):
            x = rng.uniform(-1, 1, 5)
            d = rng.uniform(-1, 1, 6)
            res.append(u.forward(x))
            res.append(u.backward(d))
            u.update(x, d, 0.05 if step != 3 else 0.0)
        u.end_minibatch()
        res.append(u.forward_noisy(np.ones(5), 0.05))
        res.append(u.get_weights().ravel())
        for m in u.members:
            res.append(m.get_weights().ravel())
        out[name] = np.concatenate(res)
    s = O.default("unitcell")  # one device, gain 1 == a plain tile with the same seed
    s.devices[0] = O.preset("reram_sb")
    u = O.unitcell(4, 3, s, 99)
    ts = O.default("tile")
    ts.device = O.preset("reram_sb")
    t = O.tile(4, 3, ts, 99)
    for _ in range(5):
        x, d = rng.uniform(-1, 1, 3), rng.uniform(-1, 1, 4)
        u.update(x, d, 0.05)
        t.update(x, d, 0.05)
    out["single"] = np.concatenate([u.get_weights().ravel(), t.get_weights().ravel()])
    return out


def inference(O):
    """program / drift_to / compensation (proj/src/inference.cpp:34-110)."""
    s = O.default("tile")
    s.device.w_max, s.device.w_min = 2.0, -2.0
    s.forward_io = O.default("perfect_io")
    t = O.tile(7, 6, s, 17)
    m = O.default("inference")
    m.prog_noise_scale, m.nu_std, m.t0, m.read_noise_scale = 0.02, 0.3, 1.0, 0.02
    target = _u(12, (7, 6), 0.5)
    w0, nu = t.program(target, m, O.rng(5).derive("program", 0))
    base = t.probe_readout(m)
    t.drift_to(w0, nu, m.t0, 1e4)
    alpha = t.drift_compensation_factor(base, m)
    return {"w0": w0, "nu": nu, "drifted": t.get_weights(), "alpha": np.array([base, alpha])}


ALL = [rng_streams, quantizer, matvec, devices, translate_trains, tile_updates, trains_apply,
       temporal, transfer, unitcell, inference]


def run_all(O) -> dict:
    out = {}
    for fn in ALL:
        for k, v in fn(O).items():
            out[f"{fn.__name__}.{k}"] = np.asarray(v)
    return out


# error cases: (description, callable(O)) -> the message must match across impls
def error_cases(O):
    def tile_bad_dims():
        O.tile(0, 3, O.default("tile"), 1)

    def tile_bad_io():
        s = O.default("tile")
        s.forward_io.dac_bits = -1
        O.tile(2, 2, s, 1)

    def tile_bad_device():
        s = O.default("tile")
        s.device.dw_min = -1.0
        O.tile(2, 2, s, 1)

    def tile_bad_bounds():
        s = O.default("tile")
        s.device.w_min = 0.5
        O.tile(2, 2, s, 1)

    def tile_bad_bl():
        s = O.default("tile")
        s.update.bl = 0
        O.tile(2, 2, s, 1)

    def tile_bad_reset():
        s = O.default("tile")
        s.temporal.reset_prob = 2.0
        O.tile(2, 2, s, 1)

    def translate_bad_lr():
        O.translate(np.ones(2), np.ones(2), -0.1, 0.001, O.default("update"))

    def translate_bad_dw():
        O.translate(np.ones(2), np.ones(2), 0.1, 0.0, O.default("update"))

    def update_negative_lr():
        O.tile(2, 2, O.default("tile"), 1).update(np.ones(2), np.ones(2), -0.5)

    def forward_nan():
        O.tile(2, 3, O.default("tile"), 1).forward(np.array([1.0, np.nan, 0.0]))

    def preset_unknown():
        O.preset("no_such_device")

    def transfer_bad_lr():
        s = O.default("transfer")
        s.transfer_lr = 0.0
        O.transfer(2, 2, s, 1)

    def unitcell_no_devices():
        s = O.default("unitcell")
        s.n_devices = 0
        O.unitcell(2, 2, s, 1)

    def unitcell_bad_gain():
        s = O.default("unitcell")
        s.gains[0] = float("inf")
        O.unitcell(2, 2, s, 1)

    def unitcell_bad_member():
        s = O.default("unitcell")
        s.n_devices = 2
        s.devices[1] = O.default("device")
        s.devices[1].dw_min = -1.0
        O.unitcell(2, 2, s, 1)

    def unitcell_zero_first_gain():
        s = O.default("unitcell")
        s.n_devices = 2
        s.devices[1] = O.default("device")
        s.gains[0], s.gains[1] = 0.0, 1.0
        O.unitcell(2, 2, s, 1).set_weights(np.ones((2, 2)))

    def drift_before_t0():
        t = O.tile(2, 2, O.default("tile"), 1)
        t.drift_to(np.zeros((2, 2)), np.zeros((2, 2)), 20.0, 19.0)

    def degenerate_comp():
        s = O.default("tile")
        s.forward_io = O.default("perfect_io")
        t = O.tile(2, 2, s, 1)
        m = O.default("inference")
        t.drift_compensation_factor(1.0, m)

    return [tile_bad_dims, tile_bad_io, tile_bad_device, tile_bad_bounds, tile_bad_bl,
            tile_bad_reset, translate_bad_lr, translate_bad_dw, update_negative_lr, forward_nan,
            preset_unknown, transfer_bad_lr, unitcell_no_devices, unitcell_bad_gain,
            unitcell_bad_member, unitcell_zero_first_gain, drift_before_t0, degenerate_comp]
