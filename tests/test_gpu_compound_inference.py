"""Tiki-Taka transfer and PCM inference on the GPU vs the oracle / the
reference's own test cases (proj/tests/test_compounds.cpp,
proj/tests/test_inference.cpp)."""
import numpy as np
import pytest

import oracle
import paper_2104_02184_b200 as xb

pytestmark = pytest.mark.gpu


def quiet_device(dw=0.001, bound=1.0):
    d = xb.default_device()
    d.dw_min, d.w_max, d.w_min = dw, bound, -bound
    return d


def ideal_transfer():
    """proj/tests/test_compounds.cpp:30-39."""
    s = xb.TransferSettings()
    s.fast_device = quiet_device()
    s.slow_device = quiet_device()
    s.forward_io = xb.perfect_io()
    s.backward_io = xb.perfect_io()
    s.transfer_every = 1
    s.transfer_lr = 0.005
    return s


@pytest.mark.parametrize("transfer_lr,exact", [(0.1, False), (0.113, True)])
def test_deterministic_transfer_matches_oracle(transfer_lr, exact):
    """test_compounds.cpp:311-358: deterministic pulses, C accumulates A's columns
    on schedule; GPU fast/slow weights vs the oracle TransferTile.  With the
    reference's own values (transfer_lr 0.1) the C counts lround(1.5) sit
    exactly on a rounding tie that the fp32 readout of A decides differently
    from the fp64 one: C may differ by one dw_min per transfer event there.
    With transfer_lr 0.113 (no ties) the GPU must match exactly."""
    s = ideal_transfer()
    s.transfer_every, s.transfer_lr = 1, transfer_lr
    s.fast_device = quiet_device(1e-4)
    s.slow_device = quiet_device(1e-4)
    s.update.pulse_type = xb.PULSE_DETERMINISTIC
    g = xb.TransferTile(2, 2, s, 17)
    O = oracle.load("restatement")
    os_ = O.default("transfer")
    for dev, src in ((os_.fast_device, s.fast_device), (os_.slow_device, s.slow_device)):
        dev.dw_min, dev.w_max, dev.w_min = src.dw_min, src.w_max, src.w_min
    os_.forward_io = O.default("perfect_io")
    os_.backward_io = O.default("perfect_io")
    os_.transfer_every, os_.transfer_lr = 1, float(np.float32(transfer_lr))
    os_.update.pulse_type = oracle.PULSE_DETERMINISTIC
    o = O.transfer(2, 2, os_, 17)
    x = np.array([0.3, -0.2], np.float32)
    d = np.array([0.25, 0.15], np.float32)
    lr = float(np.float32(0.02))
    for _ in range(6):
        g.update(x, d, lr)
        o.update(x.astype(np.float64), d.astype(np.float64), lr)
    assert g.transfer_events() == o.events() == 6
    np.testing.assert_allclose(g.fast_tile().get_weights(), o.fast.get_weights(), atol=2e-6)
    tol = 2e-6 if exact else 6 * 1e-4 + 2e-6
    np.testing.assert_allclose(g.slow_tile().get_weights(), o.slow.get_weights(), atol=tol)


def test_transfer_schedules():
    """test_compounds.cpp:247-309."""
    s = ideal_transfer()
    s.transfer_every = 3
    t = xb.TransferTile(2, 2, s, 15)
    for _ in range(10):
        t.update([1.0, 0.5], [0.8, -0.6], 0.05)
    assert t.transfer_events() == 3
    s.transfer_every = 0
    t0 = xb.TransferTile(2, 2, s, 14)
    t0.update(np.tile([1.0, 0.5], (20, 1)), np.tile([0.8, -0.6], (20, 1)), 0.05)
    assert t0.transfer_events() == 0
    assert np.all(t0.slow_tile().get_weights() == 0)
    assert np.any(t0.fast_tile().get_weights() != 0)
    s.transfer_every, s.units_in_mbatch = 1, 1
    tm = xb.TransferTile(2, 2, s, 16)
    tm.update(np.tile([1.0, 0.5], (4, 1)), np.tile([0.8, -0.6], (4, 1)), 0.05)
    assert tm.transfer_events() == 0
    tm.end_minibatch()
    assert tm.transfer_events() == 1


def test_columns_per_event():
    """test_compounds.cpp:263-283."""
    s = ideal_transfer()
    s.transfer_every, s.columns_per_event, s.transfer_lr = 1, 2, 10.0
    t = xb.TransferTile(2, 3, s, 18)
    t.fast_tile().set_weights(np.full((2, 3), 0.5))
    t.update([0.4, 0.2, 0.1], [0.3, 0.2], 1e-9)
    c = t.slow_tile().get_weights()
    assert c[0, 0] != 0 and c[0, 1] != 0 and c[0, 2] == 0


def test_expected_transfer_is_transfer_lr_times_column():
    """test_compounds.cpp:160-190 in one batch: 20000 transfer steps of column 0
    onto fresh C tiles; mean C column = transfer_lr * A column."""
    s = ideal_transfer()
    s.slow_device = quiet_device(1e-5, 1.0)
    s.transfer_lr, s.transfer_every = 0.005, 0
    t = xb.TransferTile(3, 2, s, 11)
    a = np.array([[0.05, 0.01], [-0.03, 0.04], [0.02, -0.05]], np.float32)
    t.fast_tile().set_weights(a)
    acc = np.zeros(3)
    n = 2000
    for _ in range(n):
        t.slow_tile().set_weights(np.zeros((3, 2)))
        t.transfer_step()  # column 0
        acc += t.slow_tile().get_weights()[:, 0]
        t.transfer_step()  # column 1 (cursor back to 0)
    expect = 0.005 * a[:, 0]
    assert np.all(np.abs(acc / n - expect) < 0.08 * np.abs(expect))


def test_compound_forward_mixes_gamma():
    """test_compounds.cpp:227-245."""
    for gamma, want in ((0.0, 1.0), (1.0, 2.0), (0.5, 1.5)):
        s = ideal_transfer()
        s.gamma = gamma
        t = xb.TransferTile(1, 1, s, 13)
        t.fast_tile().set_weights([[1.0]])
        t.slow_tile().set_weights([[1.0]])
        assert t.forward([1.0])[0] == pytest.approx(want, abs=1e-6)


def test_transfer_clone_is_deep_copy():
    """compound.hpp:109-111: the clone carries both members, their RNG
    positions and the transfer schedule, so identical inputs keep them equal."""
    s = xb.TransferSettings()
    s.fast_device = xb.device_preset("reram_sb")
    s.slow_device = xb.device_preset("reram_sb")
    s.transfer_every, s.gamma = 3, 0.5
    rng = np.random.default_rng(5)
    a = xb.TransferTile(16, 12, s, 41)
    a.set_weights(rng.uniform(-0.2, 0.2, (16, 12)))
    X = rng.uniform(-1, 1, (10, 12)).astype(np.float32)
    D = rng.uniform(-1, 1, (10, 16)).astype(np.float32)
    a.update(X[:4], D[:4], 0.05)
    c = a.clone()
    assert c.transfer_events() == a.transfer_events()
    a.update(X[4:], D[4:], 0.05)
    c.update(X[4:], D[4:], 0.05)
    assert c.transfer_events() == a.transfer_events() > 0
    assert np.array_equal(a.get_weights(), c.get_weights())
    assert np.array_equal(a.forward(X), c.forward(X))


def test_transfer_forward_noisy_variance():
    """compound.cpp:228-238: both members read with sigma_w = extra, so the
    output variance is extra^2 |x|^2 (1 + gamma^2) on perfect IO."""
    s = ideal_transfer()
    s.gamma = 0.5
    t = xb.TransferTile(8, 64, s, 17)
    W = np.random.default_rng(3).uniform(-0.3, 0.3, (8, 64))
    t.set_weights(W)  # C = W, A = 0
    x = np.random.default_rng(4).uniform(-1, 1, 64).astype(np.float32)
    assert np.array_equal(t.forward_noisy(x, 0.0), t.forward(x))
    Y = t.forward_noisy(np.tile(x, (4000, 1)), 0.05).astype(np.float64)
    var = 0.05 ** 2 * float(x.astype(np.float64) @ x) * (1 + 0.5 ** 2)
    exact = W @ x.astype(np.float64)
    assert np.all(np.abs(Y.mean(axis=0) - exact) < 5 * np.sqrt(var / 4000))
    assert abs(Y.var(axis=0).mean() / var - 1) < 0.06


# ------------------------------------------------------------------ inference
def wide_tile(rows, cols, seed, perfect=True):
    s = xb.TileSettings(device=quiet_device(0.001, 100.0))
    if perfect:
        s.forward_io = xb.perfect_io()
        s.backward_io = xb.perfect_io()
    return xb.AnalogTile(rows, cols, s, seed)


def quiet_model():
    m = xb.InferenceNoiseModel()
    m.prog_noise_scale = m.read_noise_scale = m.nu_mean = m.nu_std = 0.0
    m.t0 = 1.0
    return m


def test_zero_noise_program_and_frozen_drift():
    """test_inference.cpp:40-56,79-85."""
    t = wide_tile(3, 3, 1)
    target = np.random.default_rng(2).uniform(-0.5, 0.5, (3, 3)).astype(np.float32)
    t.program(target, quiet_model(), 3)
    np.testing.assert_array_equal(t.get_weights(), target)
    t.drift_to(1e8)
    np.testing.assert_array_equal(t.get_weights(), target)
    m = quiet_model()
    m.prog_noise_scale, m.prog_c0 = 1.0, 0.0
    z = wide_tile(2, 2, 4)
    z.program(np.zeros((2, 2)), m, 5)
    assert np.all(z.get_weights() == 0)


def test_programming_noise_std():
    """test_inference.cpp:58-77: 1e5 devices, std within 3 %."""
    t = wide_tile(250, 400, 6)
    m = quiet_model()
    m.prog_noise_scale = 0.1
    t.program(np.full((250, 400), 0.5), m, 7)
    dev = t.get_weights().astype(np.float64) - 0.5
    expect = 0.1 * (0.26 + 1.66 * 0.5 + 0.33 * 0.25)
    assert abs(dev.std(ddof=1) - expect) < 0.03 * expect


def test_uniform_drift_semigroup_and_errors():
    """test_inference.cpp:87-164."""
    t = wide_tile(2, 2, 11)
    m = quiet_model()
    m.nu_mean = 0.06
    target = np.random.default_rng(12).uniform(-0.5, 0.5, (2, 2)).astype(np.float32)
    t.program(target, m, 13)
    t.drift_to(100.0)
    np.testing.assert_allclose(t.get_weights(), target * 100.0 ** -0.06, atol=1e-6)
    with pytest.raises(xb.Error, match="drift_to: t < t0"):
        t.drift_to(0.5)
    a, b = wide_tile(3, 3, 17), wide_tile(3, 3, 17)
    m.nu_mean, m.nu_std = 0.08, 0.5
    tg = np.random.default_rng(18).uniform(-0.5, 0.5, (3, 3))
    a.program(tg, m, 19)
    b.program(tg, m, 19)
    a.drift_to(1e3)
    a.drift_to(1e6)
    b.drift_to(1e6)
    np.testing.assert_array_equal(a.get_weights(), b.get_weights())  # w0-based: exact semigroup
    # sign preservation (test_inference.cpp:145-164)
    s = wide_tile(4, 4, 20)
    m.nu_mean, m.nu_std = 0.1, 0.3
    tg = np.where((np.add.outer(np.arange(4), np.arange(4)) % 2) == 0, 0.5, -0.5)
    s.program(tg, m, 21)
    s.drift_to(1e6)
    assert np.all(s.get_weights() * tg > 0)


def test_drift_slope_recovers_nu():
    """test_inference.cpp:250-294 / acceptance criterion 5."""
    t = wide_tile(100, 100, 37)
    m = quiet_model()
    m.nu_mean, m.nu_std = 0.06, 0.3
    t.program(np.full((100, 100), 0.5), m, 38)
    times = [1.0, 10.0, 100.0, 1000.0]
    snaps = []
    for tt in times:
        t.drift_to(tt)
        snaps.append(np.log(t.get_weights().astype(np.float64)))
    lt = np.log(times)
    slope = -np.polyfit(lt, np.stack([s.ravel() for s in snaps]), 1)[0]
    assert abs(slope.mean() - 0.06) < 0.05 * 0.06


def test_compensation_factor():
    """test_inference.cpp:207-222: alpha = 1 at t0 and (t/t0)^nu under uniform drift."""
    t = wide_tile(3, 3, 29)
    m = quiet_model()
    m.nu_mean = 0.06
    t.program(np.random.default_rng(30).uniform(-0.5, 0.5, (3, 3)), m, 31)
    base = t.probe_readout(m)
    assert t.drift_compensation_factor(base, m) == pytest.approx(1.0, rel=1e-6)
    t.drift_to(100.0)
    assert abs(t.drift_compensation_factor(base, m) - 100.0 ** 0.06) < 1e-5
    z = wide_tile(2, 2, 36)
    with pytest.raises(xb.Error, match="degenerate readout"):
        z.drift_compensation_factor(1.0, m)


@pytest.mark.parametrize("exact_io", [False, True])
def test_transfer_step_equals_explicit_read_and_update(exact_io):
    """The device-side transfer (column gather + the shared output stage,
    then a pulsed update restricted to column j's block, no host round trip)
    is bit for bit the reference's definition run through the public API on
    a clone: A.forward_with_io(e_j, transfer io) then C.update(e_j, readout,
    transfer_lr) (proj/src/compound.cpp:257-267), noise on."""
    s = xb.TransferSettings()
    s.fast_device = xb.device_preset("reram_sb")
    s.slow_device = xb.device_preset("reram_sb")
    s.transfer_lr = 0.3
    if exact_io:  # perfect transfer io (no converters)
        s.has_transfer_io = 1
        s.transfer_io = xb.perfect_io()
    d_out, d_in = 300, 70
    t = xb.TransferTile(d_out, d_in, s, 12)
    r = np.random.default_rng(3)
    t.fast_tile().set_weights(r.uniform(-0.3, 0.3, (d_out, d_in)).astype(np.float32))
    t.slow_tile().set_weights(r.uniform(-0.3, 0.3, (d_out, d_in)).astype(np.float32))
    c = t.clone()
    io = s.transfer_io if exact_io else s.forward_io
    for j in range(3):
        t.transfer_step()
        e = np.zeros(d_in, np.float32)
        e[j] = 1.0
        ro = c.fast_tile().forward_with_io(e, io)
        c.slow_tile().update(e, ro, s.transfer_lr)
    np.testing.assert_array_equal(t.slow_tile().get_weights(), c.slow_tile().get_weights())
    np.testing.assert_array_equal(t.fast_tile().get_weights(), c.fast_tile().get_weights())
    # the next forward of A draws the same noise on both (read counters in step)
    X = r.uniform(-1, 1, (4, d_in)).astype(np.float32)
    np.testing.assert_array_equal(t.fast_tile().forward(X), c.fast_tile().forward(X))
