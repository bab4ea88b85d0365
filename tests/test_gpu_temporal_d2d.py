"""Temporal processes (decay, diffusion, reset; proj/src/tile.cpp:128-156) and
the device-to-device realization (proj/src/device.cpp:26-46) on the GPU tile,
re-running the reference's own cases (proj/tests/test_tile.cpp:307-404,
proj/tests/test_devices.cpp:33-47) through the C ABI.  The draws are Philox
(not the reference's mt19937), so the random cases are checked against the
same statistical oracles the reference uses; the deterministic ones against
the closed forms (fp32 weights: relative tolerance 2e-6 instead of 1e-12)."""
import numpy as np
import pytest

import paper_2104_02184_b200 as xb

pytestmark = pytest.mark.gpu


def quiet_settings(dw_min=0.001, bound=1.0):  # proj/tests/helpers.hpp:70-86
    dev = xb.default_device()
    dev.kind, dev.dw_min, dev.w_max, dev.w_min = xb.CONSTANT_STEP, dw_min, bound, -bound
    return xb.TileSettings(device=dev, forward_io=xb.io_off(), backward_io=xb.io_off())


def random_matrix(r, c, scale, seed):
    return np.random.default_rng(seed).uniform(-scale, scale, (r, c)).astype(np.float32)


def temporal(**kw):
    tp = xb.TemporalParams()
    for k, v in kw.items():
        setattr(tp, k, v)
    return tp


def test_all_zero_temporal_parameters_are_the_identity():  # test_tile.cpp:307-314
    t = xb.AnalogTile(3, 3, quiet_settings(), 13)
    t.set_weights(random_matrix(3, 3, 0.5, 71))
    before = t.get_weights()
    t.apply_temporal_step(temporal())
    t.end_minibatch()
    np.testing.assert_array_equal(t.get_weights(), before)


def test_decay_follows_closed_form():  # test_tile.cpp:316-334
    t = xb.AnalogTile(2, 2, quiet_settings(), 14)
    t.set_weights(random_matrix(2, 2, 0.5, 81))
    w = t.get_weights().astype(np.float64)
    tp = temporal(decay_rate=0.1)
    for _ in range(7):
        t.apply_temporal_step(tp)
    np.testing.assert_allclose(t.get_weights(), w * 0.9 ** 7, rtol=2e-6)


def test_decay_through_end_minibatch_settings():
    """end_minibatch applies the tile's own TemporalParams (tile.hpp:99-100)."""
    s = quiet_settings()
    s.temporal.decay_rate = 0.2
    t = xb.AnalogTile(8, 8, s, 3)
    w = random_matrix(8, 8, 0.5, 4)
    t.set_weights(w)
    t.end_minibatch()
    t.end_minibatch()
    np.testing.assert_allclose(t.get_weights(), w.astype(np.float64) * 0.8 ** 2, rtol=2e-6)


def test_diffusion_variance_grows_like_n_sigma2():  # test_tile.cpp:336-356
    t = xb.AnalogTile(50, 50, quiet_settings(0.001, 100.0), 15)
    tp = temporal(diffusion_sigma=0.01)
    for _ in range(20):
        t.apply_temporal_step(tp)
    w = t.get_weights().astype(np.float64).ravel()
    expect = 20 * 0.01 ** 2
    assert abs(w.var(ddof=1) - expect) < 0.15 * expect
    assert abs(w.mean()) < 5 * np.sqrt(expect / w.size)


def test_reset_empties_devices_at_the_configured_rate():  # test_tile.cpp:358-387
    t = xb.AnalogTile(40, 40, quiet_settings(), 16)
    t.set_weights(np.full((40, 40), 0.5, np.float32))
    t.apply_temporal_step(temporal(reset_prob=1.0))
    assert np.all(t.get_weights() == 0.0)
    t2 = xb.AnalogTile(40, 40, quiet_settings(), 17)
    t2.set_weights(np.full((40, 40), 0.5, np.float32))
    t2.apply_temporal_step(temporal(reset_prob=0.3))
    frac = np.mean(t2.get_weights() == 0.0)
    assert 0.25 < frac < 0.35
    assert np.all((t2.get_weights() == 0.0) | (t2.get_weights() == 0.5))


def test_temporal_variation_draws_are_fixed_per_device():  # test_tile.cpp:389-404
    s = quiet_settings(0.001, 100.0)
    a, b = xb.AnalogTile(4, 4, s, 18), xb.AnalogTile(4, 4, s, 18)
    w = random_matrix(4, 4, 0.5, 91)
    a.set_weights(w)
    b.set_weights(w)
    tp = temporal(decay_rate=0.05, decay_dtod=0.5)
    a.apply_temporal_step(tp)
    b.apply_temporal_step(tp)
    np.testing.assert_array_equal(a.get_weights(), b.get_weights())


def test_decay_d2d_spread_and_mean():
    """decay_dtod: per-cell rates r (1 + dtod xi), xi fixed per device and
    clamped to [0, 1] (tile.cpp:136-139): the per-cell factor w'/w has mean
    1 - r and spread r dtod, and repeats identically on the next step."""
    s = quiet_settings(0.001, 100.0)
    t = xb.AnalogTile(100, 100, s, 21)
    w = np.full((100, 100), 0.5, np.float32)
    t.set_weights(w)
    tp = temporal(decay_rate=0.1, decay_dtod=0.3)
    t.apply_temporal_step(tp)
    f1 = t.get_weights().astype(np.float64) / 0.5
    t.apply_temporal_step(tp)
    f2 = t.get_weights().astype(np.float64) / (0.5 * f1)
    assert abs(f1.mean() - 0.9) < 5 * 0.03 / 100
    assert abs(f1.std() / 0.03 - 1) < 0.05
    np.testing.assert_allclose(f2, f1, rtol=1e-5)  # the same device rates again


def test_weights_stay_within_device_bounds_after_diffusion():
    """Every temporal write clips to the per-cell bounds (tile.cpp:153)."""
    t = xb.AnalogTile(30, 30, quiet_settings(0.001, 0.05), 5)
    t.apply_temporal_step(temporal(diffusion_sigma=0.2))
    w = t.get_weights()
    assert np.abs(w).max() <= 0.05 + 1e-7
    assert np.mean(np.abs(w) == np.float32(0.05)) > 0.5


def test_device_to_device_spread_reproduces_the_configured_moment():  # test_devices.cpp:33-47
    dev = xb.default_device()
    dev.kind, dev.dw_min, dev.w_max, dev.w_min = xb.CONSTANT_STEP, 0.002, 0.6, -0.6
    dev.dw_min_dtod = 0.3
    t = xb.AnalogTile(100, 100, xb.TileSettings(device=dev), 2)
    up, down, wmax, wmin = t.get_device()
    up = up.astype(np.float64).ravel()
    assert abs(up.std(ddof=1) / up.mean() - 0.3) < 0.03
    assert abs(up.mean() - 0.002) < 5 * 0.3 * 0.002 / 100
    np.testing.assert_array_equal(up, down.ravel())  # up_down = up_down_dtod = 0
    assert np.all(wmax == np.float32(0.6)) and np.all(wmin == np.float32(-0.6))


def test_realization_floors_and_bound_spreads():
    """device.cpp:34-42: dw >= 0.01 dw_min, w_max >= 0.01 w_max, w_min <=
    0.01 w_min; bias spread up_down_dtod; bound spreads w_*_dtod."""
    dev = xb.device_preset("reram_sb")
    dev.dw_min_dtod = 2.0  # a wide spread exercises the floors
    dev.w_max_dtod = dev.w_min_dtod = 0.2
    t = xb.AnalogTile(120, 120, xb.TileSettings(device=dev), 9)
    up, down, wmax, wmin = (a.astype(np.float64).ravel() for a in t.get_device())
    floor = 0.01 * dev.dw_min
    assert up.min() >= floor * (1 - 1e-6) and down.min() >= floor * (1 - 1e-6)
    # dw = max(dw_min (1 + 2 xi), floor) is floored where xi < -0.495, P = 0.310;
    # the up/down bias (+-1 %) then moves one of the two just above the floor
    from math import erf, sqrt
    p = 0.5 * (1 + erf(-0.495 / sqrt(2)))
    frac = np.mean(np.minimum(up, down) <= floor * (1 + 1e-6))
    assert abs(frac - p) < 5 * np.sqrt(p * (1 - p) / up.size)
    assert wmax.min() >= 0.006 * (1 - 1e-6) and wmin.max() <= -0.006 * (1 - 1e-6)
    assert abs(wmax.std() / 0.6 - 0.2) < 0.02 and abs(wmin.std() / 0.6 - 0.2) < 0.02
    # up/down asymmetry: up = dw (1 + b), down = dw (1 - b), b ~ N(0, 0.01)
    ok = (up > floor * 1.01) & (down > floor * 1.01)
    b = (up[ok] - down[ok]) / (up[ok] + down[ok])
    assert abs(b.std() - 0.01) < 0.002 and abs(b.mean()) < 5 * 0.01 / np.sqrt(ok.sum())
