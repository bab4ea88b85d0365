"""Pulsed-update parity: the CUDA path (through the C ABI) vs the CPU oracle.

Protocols:
  (i)   noise off, identical trains: GPU-generated packed trains are unpacked
        and fed to the oracle's apply_pulse_trains; coincidence counts must be
        bit-exact and weights within 1e-5 relative;
  (ii)  noise off, deterministic_implicit mode: the whole update is RNG-free;
  (iii) noise on: per-pulse moments and E[dW] = lr d x^T within confidence
        bounds;
plus the reference's own known-answer and edge-case tests.
"""
import numpy as np
import pytest

import oracle
import paper_2104_02184_b200 as xb
from paper_2104_02184_b200 import trains as T
from gpu_helpers import apply_words_to_oracle, close, twin

pytestmark = pytest.mark.gpu

LAWS = [xb.CONSTANT_STEP, xb.LINEAR_STEP, xb.SOFT_BOUNDS, xb.EXP_STEP]


def cfg_law(kind, dw=0.002, dtod=0.3, std=0.0, blm=0, bl=31):
    dev = xb.default_device()
    dev.kind, dev.dw_min, dev.dw_min_dtod, dev.dw_min_std = kind, dw, dtod, std
    dev.w_max, dev.w_min, dev.up_down, dev.up_down_dtod = 0.6, -0.6, 0.05, 0.01
    dev.w_max_dtod = dev.w_min_dtod = 0.1
    dev.slope, dev.gamma = 0.8, 2.0
    c = xb.TileSettings(device=dev)
    c.update.bl, c.update.bl_management = bl, blm
    return c


def rand_xd(B, d_in, d_out, seed):
    r = np.random.default_rng(seed)
    return (r.uniform(-1, 1, (B, d_in)).astype(np.float32),
            r.uniform(-1, 1, (B, d_out)).astype(np.float32))


@pytest.mark.parametrize("kind", LAWS)
@pytest.mark.parametrize("shape", [(37, 45), (64, 96)])
def test_identical_trains_parity(kind, shape):
    """Protocol (i) for every law, d2d on, BL management on, B = 24."""
    d_out, d_in = shape
    cfg = cfg_law(kind, blm=1)
    g, o = twin(cfg, d_out, d_in, seed=11 + kind)
    X, D = rand_xd(24, d_in, d_out, 5)
    lr = np.full(24, 0.02, np.float32)
    xw, dw, bl = g.generate_trains(X, D, lr)
    g.apply_pulse_trains(xw, dw)
    apply_words_to_oracle(o, xw, dw, bl)
    wg, wo = g.get_weights(), o.get_weights()
    ok = close(wg, wo, 1e-5, 0.1)
    assert ok.all(), f"max |dw| {np.max(np.abs(wg - wo))} at {np.argwhere(~ok)[:3]}"
    assert np.any(wg != np.random.default_rng(3).uniform(-0.1, 0.1, shape).astype(np.float32))


@pytest.mark.parametrize("kind", LAWS)
@pytest.mark.parametrize("B", [40, 13])
def test_update_equals_generate_plus_apply(kind, B):
    """The fused update path draws exactly the trains generate_trains reports
    (B = 13: partial 4-sample quads of the x train layout)."""
    cfg = cfg_law(kind, std=0.3)
    a = xb.AnalogTile(50, 70, cfg, 9)
    a.set_weights(np.random.default_rng(2).uniform(-0.2, 0.2, (50, 70)))
    b = a.clone()
    X, D = rand_xd(B, 70, 50, 6)
    xw, dw, bl = b.generate_trains(X, D, 0.01)
    a.update(X, D, 0.01)
    b.apply_pulse_trains(xw, dw)
    np.testing.assert_array_equal(a.get_weights(), b.get_weights())


def test_coincidence_counts_bit_exact():
    """proj/tests/test_pulsed.cpp:133-158 at scale: a power-of-two step makes
    every weight change an exact multiple of dw_min, so W / dw_min recovers
    the coincidence counts, which must equal the brute-force AND/popcount of
    the packed trains and the oracle's slot-major triple loop."""
    dw_min = 2.0 ** -12
    dev = xb.default_device()
    dev.dw_min, dev.w_max, dev.w_min = dw_min, 64.0, -64.0
    cfg = xb.TileSettings(device=dev)
    d_out, d_in, B = 96, 160, 1
    g, o = twin(cfg, d_out, d_in, w_scale=0.0)
    for trial in range(3):
        X, D = rand_xd(B, d_in, d_out, 100 + trial)
        xw, dw, bl = g.generate_trains(X, D, 0.05)
        before_g = g.get_weights().astype(np.float64)
        before_o = o.get_weights()
        g.apply_pulse_trains(xw, dw)
        apply_words_to_oracle(o, xw, dw, bl)
        dg = (g.get_weights().astype(np.float64) - before_g) / dw_min
        do = (o.get_weights() - before_o) / dw_min
        brute = T.coincidences(xw[0], dw[0]).astype(np.int64)
        sign = np.where(((dw[0][:, None] ^ xw[0][None, :]) >> 31) == 0, 1, -1)
        np.testing.assert_array_equal(dg, brute * sign)
        np.testing.assert_array_equal(do, brute * sign)
        assert brute.sum() > 100


def test_translate_and_bl_management_match_oracle():
    """Per-sample bl (BL management) and train statistics follow the oracle's
    translate() on the same fp32 inputs (proj/src/pulsed.cpp:25-66)."""
    O = oracle.load("restatement")
    cfg = cfg_law(xb.CONSTANT_STEP, dw=0.001, dtod=0.0, blm=1)
    g = xb.AnalogTile(40, 30, cfg, 1)
    X, D = rand_xd(64, 30, 40, 8)
    X[3] *= 0.01
    D[5] *= 0.02
    lr = np.full(64, 0.001, np.float32)
    lr[7] = 0.0
    xw, dw, bl = g.generate_trains(X, D, lr)
    up = O.default("update")
    up.bl, up.bl_management = 31, 1
    for b in range(64):
        if lr[b] == 0:
            assert bl[b] == 0 and not xw[b].any() and not dw[b].any()
            continue
        obl, px, pd, sx, sd = O.translate(X[b].astype(np.float64), D[b].astype(np.float64),
                                          float(lr[b]), 0.001, up)
        assert bl[b] == obl
        # no bits at or beyond bl, signs as the oracle's
        assert not np.any((xw[b] & 0x7FFFFFFF) >> obl)
        _, gsx = T.unpack(xw[b], obl)
        nz = sx != 0
        np.testing.assert_array_equal(gsx[nz], sx[nz])


def test_train_bits_are_bernoulli_p():
    """Slot counts are Binomial(bl, p) with the oracle's p (test_pulsed.cpp:81-108)."""
    O = oracle.load("restatement")
    cfg = cfg_law(xb.CONSTANT_STEP, dw=0.001, dtod=0.0)
    d_in, d_out, B = 8, 8, 4096
    g = xb.AnalogTile(d_out, d_in, cfg, 4)
    x = np.array([1.0, -0.8, 0.6, 0.4, 0.2, -0.1, 0.05, 0.0], np.float32)
    d = np.array([0.9, -0.7, 0.5, 0.3, 0.1, 0.05, -0.02, 0.01], np.float32)
    X = np.tile(x, (B, 1))
    D = np.tile(d, (B, 1))
    xw, dw, bl = g.generate_trains(X, D, 0.01)
    up = O.default("update")
    _, px, pd, _, _ = O.translate(x.astype(np.float64), d.astype(np.float64), 0.01, 0.001, up)
    for words, p in ((xw, px), (dw, pd)):
        counts = np.array([[bin(int(v) & 0x7FFFFFFF).count("1") for v in row] for row in words])
        mean = counts.mean(axis=0)
        se = np.sqrt(31 * p * (1 - p) / B) + 1e-12
        assert np.all(np.abs(mean - 31 * p) <= 4.5 * se), (mean, 31 * p)
    # x == 0 line never fires and carries sign 0 (no sign bit)
    assert not np.any(xw[:, 7])


@pytest.mark.parametrize("kind", LAWS)
def test_deterministic_mode_parity(kind):
    """Protocol (ii): deterministic_implicit update is RNG-free; counts are
    lround(bl p_d p_x) in fp64 on both sides (proj/src/pulsed.cpp:128-144)."""
    cfg = cfg_law(kind, blm=1)
    cfg.update.pulse_type = xb.PULSE_DETERMINISTIC
    g, o = twin(cfg, 33, 41, seed=21)
    X, D = rand_xd(12, 41, 33, 12)
    lr = float(np.float32(0.05))  # the GPU receives fp32 learning rates
    g.update(X, D, lr)
    for b in range(12):
        o.update(X[b].astype(np.float64), D[b].astype(np.float64), lr)
    ok = close(g.get_weights(), o.get_weights(), 1e-5, 0.1)
    assert ok.all(), np.max(np.abs(g.get_weights() - o.get_weights()))


def test_saturated_trains_kat():
    """proj/tests/test_pulsed.cpp:66-79: saturated probabilities, -31 dw_min exactly."""
    dev = xb.default_device()
    dev.dw_min = 0.001
    g = xb.AnalogTile(1, 1, xb.TileSettings(device=dev, forward_io=xb.io_off(),
                                            backward_io=xb.io_off()), 2)
    g.update([1.0], [-1.0], 10.0)
    assert g.get_weights()[0, 0] == pytest.approx(-31 * 0.001, rel=1e-6)


def test_disjoint_trains_leave_weights_unchanged():
    """proj/tests/test_pulsed.cpp:110-131."""
    g = xb.AnalogTile(2, 2, xb.TileSettings(), 4)
    g.set_weights(np.random.default_rng(5).uniform(-0.3, 0.3, (2, 2)))
    before = g.get_weights()
    even = sum(1 << t for t in range(0, 10, 2))
    odd = sum(1 << t for t in range(1, 10, 2))
    g.apply_pulse_trains(np.array([[even, even]], np.uint32), np.array([[odd, odd]], np.uint32))
    np.testing.assert_array_equal(g.get_weights(), before)


def test_noop_updates():
    """proj/tests/test_pulsed.cpp:177-189 and zero columns (:191-201)."""
    g = xb.AnalogTile(2, 2, xb.TileSettings(), 11)
    g.set_weights(np.random.default_rng(12).uniform(-0.3, 0.3, (2, 2)))
    before = g.get_weights()
    g.update([[1, 1], [0, 0], [1, 1]], [[1, 1], [1, 1], [0, 0]], [0.0, 0.1, 0.1])
    np.testing.assert_array_equal(g.get_weights(), before)
    t = xb.AnalogTile(2, 2, xb.TileSettings(), 13)
    X = np.tile(np.array([0.8, 0.0], np.float32), (100, 1))
    D = np.tile(np.array([0.7, -0.4], np.float32), (100, 1))
    t.update(X, D, 0.05)
    w = t.get_weights()
    assert w[0, 1] == 0.0 and w[1, 1] == 0.0 and w[0, 0] != 0.0


def test_errors_match_reference():
    g = xb.AnalogTile(2, 3, xb.TileSettings(), 12)
    with pytest.raises(xb.Error, match="translate: learning rate must be > 0"):
        g.update([1.0, 1.0, 1.0], [1.0, 1.0], -0.5)
    with pytest.raises(xb.Error, match="update\\(x\\): non-finite entry"):
        g.update([1.0, np.nan, 1.0], [1.0, 1.0], 0.1)
    with pytest.raises(xb.Error, match="forward: length 2, expected 3"):
        g.forward([1.0, 2.0])
    with pytest.raises(xb.Error, match="forward: non-finite entry"):
        g.forward([1.0, np.inf, 0.0])
    with pytest.raises(xb.Error, match="learning_rate: must be > 0"):
        g.set_learning_rate(0.0)
    with pytest.raises(xb.Error, match="set_weights: shape"):
        g.set_weights(np.zeros((3, 2)))
    bad = xb.TileSettings()
    bad.device.dw_min = -1
    with pytest.raises(xb.Error, match="device.dw_min: must be > 0"):
        xb.AnalogTile(2, 2, bad, 1)
    with pytest.raises(xb.Error, match="tile: dimensions must be >= 1"):
        xb.AnalogTile(0, 2, xb.TileSettings(), 1)


@pytest.mark.parametrize("shape", [(64, 1024, 8), (37, 101, 5), (600, 96, 120), (96, 600, 120)])
def test_nonfinite_inputs_leave_tile_untouched(shape):
    """check_input (tile.cpp:65-75): an Inf/NaN anywhere (16-B vector body or
    scalar tail, x or d) raises before the weights or the noise streams move.
    Calls up to 2^16 input floats are scanned on the host before the copy;
    larger ones on the device after it (the last two shapes: the update, and
    the backward or the forward, take the device path)."""
    R, C, B = shape
    rng = np.random.default_rng(3)
    X = rng.uniform(-1, 1, (B, C)).astype(np.float32)
    D = rng.uniform(-1, 1, (B, R)).astype(np.float32)
    w0 = rng.uniform(-0.1, 0.1, (R, C)).astype(np.float32)
    s = xb.TileSettings(device=xb.device_preset("reram_sb"))
    a, b = xb.AnalogTile(R, C, s, 21), xb.AnalogTile(R, C, s, 21)
    a.set_weights(w0)
    b.set_weights(w0)
    for arr, pos, val, msg in ((X, (B - 1, C - 1), np.nan, "update\\(x\\)"),
                               (D, (B // 2, 3), np.inf, "update\\(d\\)"),
                               (D, (B - 1, R - 1), -np.inf, "update\\(d\\)")):
        bad = arr.copy()
        bad[pos] = val
        args = (bad, D) if arr is X else (X, bad)
        with pytest.raises(xb.Error, match=msg + ": non-finite entry"):
            a.update(*args, 0.01)
    Xb = X.copy()
    Xb[0, C // 2] = np.nan
    with pytest.raises(xb.Error, match="forward: non-finite entry"):
        a.forward(Xb)
    Db = D.copy()
    Db[B - 1, R - 1] = np.inf
    with pytest.raises(xb.Error, match="backward: non-finite entry"):
        a.backward(Db)
    assert np.array_equal(a.get_weights(), b.get_weights())
    a.update(X, D, 0.01)
    b.update(X, D, 0.01)
    assert np.array_equal(a.get_weights(), b.get_weights())
    assert np.array_equal(a.forward(X), b.forward(X))
    assert np.array_equal(a.backward(D), b.backward(D))


def test_mean_update_equals_lr_d_xT():
    """Acceptance criterion 2 / test_pulsed.cpp:203-231: E[dW] = lr d x^T within
    2 %.  2048 samples of the same (x, d) in one batched call on a ConstantStep
    tile far from its bounds: the accumulated change / 2048 estimates E[dW];
    256 column replicas of each x_j tighten the x-train average."""
    dev = xb.default_device()
    dev.dw_min, dev.w_max, dev.w_min = 0.001, 1000.0, -1000.0
    cfg = xb.TileSettings(device=dev)
    reps, B = 256, 2048
    x = np.array([1.0, -0.8, 0.6, 0.4], np.float32)
    d = np.array([0.9, -0.7, 0.5, 0.3], np.float32)
    g = xb.AnalogTile(4, 4 * reps, cfg, 2001)
    lr = 0.01
    g.update(np.tile(np.tile(x, reps), (B, 1)), np.tile(d, (B, 1)), lr)
    w = g.get_weights().astype(np.float64).reshape(4, reps, 4).mean(axis=1) / B
    expect = lr * np.outer(d, x)
    mask = np.abs(np.outer(d, x)) > 0.1
    rel = np.abs(w - expect)[mask] / np.abs(expect)[mask]
    assert rel.max() < 0.02, rel


def test_c2c_noise_moments():
    """Per-pulse dW under cycle-to-cycle noise: mean dw_min, std dw_min_std
    dw_min (proj/tests/test_devices.cpp:163-176), from saturated trains on a
    ConstantStep tile far from the bounds: after k pulses the change is
    sum of k independent dw (1 + std xi)."""
    dev = xb.default_device()
    dev.dw_min, dev.dw_min_std, dev.w_max, dev.w_min = 0.001, 0.3, 10.0, -10.0
    g = xb.AnalogTile(64, 1024, xb.TileSettings(device=dev), 77)
    n = 64 * 1024
    full = np.uint32((1 << 31) - 1)
    g.apply_pulse_trains(np.full((1, 1024), full, np.uint32), np.full((1, 64), full, np.uint32))
    dw = g.get_weights().ravel().astype(np.float64)
    k = 31
    mean, var = dw.mean(), dw.var(ddof=1)
    se_mean = np.sqrt(k * (0.3 * 0.001) ** 2 / n)
    assert abs(mean - k * 0.001) < 4 * se_mean
    expect_var = k * (0.3 * 0.001) ** 2
    assert abs(var / expect_var - 1) < 4 * np.sqrt(2 / (n - 1))


@pytest.mark.parametrize("kind", [xb.CONSTANT_STEP, xb.LINEAR_STEP, xb.SOFT_BOUNDS, xb.EXP_STEP])
def test_c2c_single_pulse_distribution(kind):
    """One pulse per cell from w = 0: dW / h - 1 = std z with h the law's
    step at w = 0 (dw_min for ConstantStep), so the 262 144 cells sample the
    c2c factor directly.  z must be a standard normal: mean, variance,
    skewness and kurtosis within 5 standard errors, and a Kolmogorov-Smirnov
    distance below 5/sqrt(n) (the 16-bit radius and the 256-angle
    Box-Muller grid are invisible at this sample size)."""
    from math import erf, sqrt
    dev = xb.default_device()
    dev.kind = kind
    dev.dw_min, dev.dw_min_std, dev.w_max, dev.w_min = 2.0 ** -10, 0.25, 10.0, -10.0
    h = dev.dw_min  # ConstantStep, and LinearStep / SoftBounds at w = 0
    if kind == xb.LINEAR_STEP:
        dev.slope = 0.5
    if kind == xb.EXP_STEP:
        dev.gamma = 2.0
        h = dev.dw_min * np.exp(-dev.gamma * (0.0 - dev.w_min) / (dev.w_max - dev.w_min))
    R, C = 256, 1024
    g = xb.AnalogTile(R, C, xb.TileSettings(device=dev, weight_precision=xb.W_FP32), 91)
    g.apply_pulse_trains(np.ones((1, C), np.uint32), np.ones((1, R), np.uint32))  # slot 0 only
    z = (g.get_weights().ravel().astype(np.float64) / h - 1.0) / dev.dw_min_std
    n = z.size
    assert abs(z.mean()) < 5 / np.sqrt(n)
    assert abs(z.var() - 1) < 5 * np.sqrt(2 / n)
    assert abs(((z - z.mean()) ** 3).mean() / z.std() ** 3) < 5 * np.sqrt(6 / n)
    assert abs(((z - z.mean()) ** 4).mean() / z.var() ** 2 - 3) < 5 * np.sqrt(24 / n)
    zs = np.sort(z)
    cdf = 0.5 * (1 + np.vectorize(erf)(zs / sqrt(2)))
    ks = np.max(np.maximum(np.arange(1, n + 1) / n - cdf, cdf - np.arange(n) / n))
    assert ks < 5 / np.sqrt(n), ks


def test_softbounds_closed_form_on_gpu():
    """Acceptance criterion 3 through the tile: 31 up pulses per call on a
    noise-free SoftBounds cell follow w_n = w_max - w_max (1 - dw/w_max)^n."""
    dev = xb.default_device()
    dev.kind, dev.dw_min, dev.w_max, dev.w_min = xb.SOFT_BOUNDS, 0.01, 0.6, -0.6
    g = xb.AnalogTile(1, 1, xb.TileSettings(device=dev), 3001)
    full = np.uint32((1 << 31) - 1)
    worst = 0.0
    for call in range(1, 33):
        g.apply_pulse_trains(np.array([[full]]), np.array([[full]]))
        n = 31 * call
        closed = 0.6 - 0.6 * (1 - 0.01 / 0.6) ** n
        worst = max(worst, abs(float(g.get_weights()[0, 0]) - closed))
    assert worst <= 2e-6


def test_bounds_respected_all_laws():
    """proj/tests/test_devices.cpp:125-148 under heavy c2c noise."""
    for kind in LAWS:
        dev = xb.default_device()
        dev.kind, dev.dw_min, dev.dw_min_dtod, dev.dw_min_std = kind, 0.05, 0.3, 0.5
        dev.w_max, dev.w_min, dev.w_max_dtod, dev.w_min_dtod = 0.4, -0.5, 0.2, 0.2
        g = xb.AnalogTile(32, 64, xb.TileSettings(device=dev), 6)
        X, D = rand_xd(64, 64, 32, 9)
        g.update(X, D, 1.0)
        w = g.get_weights()
        _, _, wmax, wmin = g.get_device()
        assert np.all(w <= wmax) and np.all(w >= wmin)


def test_batched_chunks_beyond_smem_batch():
    """B larger than the kernel's staged chunk (256 samples) equals two calls
    (noise off: the c2c counter is the only call-dependent state)."""
    cfg = cfg_law(xb.SOFT_BOUNDS)
    a = xb.AnalogTile(40, 64, cfg, 5)
    a.set_weights(np.random.default_rng(1).uniform(-0.1, 0.1, (40, 64)))
    b = a.clone()
    X, D = rand_xd(600, 64, 40, 2)
    xw, dw, bl = a.generate_trains(X, D, 0.01)
    a.apply_pulse_trains(xw, dw)
    b.apply_pulse_trains(xw[:256], dw[:256])
    b.apply_pulse_trains(xw[256:], dw[256:])
    np.testing.assert_array_equal(a.get_weights(), b.get_weights())


@pytest.mark.parametrize("wp", [xb.W_AUTO, xb.W_FP32X2, xb.W_FP32])
def test_compensated_weights_track_fp64(restatement, wp):
    """SURVEY §7 hard part 3: the "ideal" preset steps by dw_min = 1e-6, only
    ~17 fp32 ulps of w = 0.5, so fp32 storage rounds every pulse the same way
    and drifts.  Compensated storage (auto-selected for such devices) adds each
    step error-free and lands on the reference's fp64 result."""
    dev = xb.device_preset("ideal")
    s = xb.TileSettings(device=dev, weight_precision=wp)
    t = xb.AnalogTile(4, 8, s, 5)
    t.set_weights(np.full((4, 8), 0.5))
    n = 2000  # saturated trains: 31 up pulses per sample
    X = np.ones((n, 8), np.float32)
    D = np.ones((n, 4), np.float32)
    t.update(X, D, 1e-3)
    # the reference's ConstantStep in fp64: every pulse adds dw_min exactly
    ts = restatement.default("tile")
    ts.device = restatement.preset("ideal")
    o = restatement.tile(4, 8, ts, 5)
    o.set_weights(np.full((4, 8), 0.5))
    for b in range(0, n, 500):  # a quarter of the samples through the oracle
        o.update(np.ones(8), np.ones(4), 1e-3)
    assert np.allclose(o.get_weights(), 0.5 + 31 * 4 * dev.dw_min, atol=1e-12)
    want = 0.5 + 31 * n * dev.dw_min
    got = t.get_weights().astype(np.float64)
    if wp == xb.W_FP32:
        assert np.abs(got - want).max() > 1e-4  # the drift the compensation removes
    else:
        assert np.abs(got - want).max() < 2e-7, np.abs(got - want).max()
