"""UnitCellTile on the GPU (proj/src/compound.cpp:12-174) against the oracle
and the reference's own unit-cell tests (proj/tests/test_compounds.cpp:43-150).

The GPU draws its trains from Philox, so RNG-dependent results are compared
by structure (which member moved, by how much per coincidence) and in
expectation; RNG-free paths (set/get, perfect-IO forward/backward, errors)
are compared with the oracle directly."""
import numpy as np
import pytest

import oracle
import paper_2104_02184_b200 as xb

pytestmark = pytest.mark.gpu


def const_dev(dw=2.0 ** -10, bound=8.0):
    d = xb.default_device()
    d.dw_min, d.w_max, d.w_min = dw, bound, -bound
    return d


def cell(devices, gains, policy, io=None, seed=7, shape=(6, 5)):
    io = io if io is not None else xb.perfect_io()
    s = xb.UnitCellSettings(devices, gains, policy, forward_io=io, backward_io=io)
    return xb.UnitCellTile(shape[0], shape[1], s, seed)


def oracle_cell(O, devices, gains, policy, seed=7, shape=(6, 5)):
    s = O.default("unitcell")
    s.n_devices, s.policy = len(devices), policy
    for k, (d, g) in enumerate(zip(devices, gains)):
        od = O.default("device")
        for f in ("kind", "dw_min", "dw_min_dtod", "dw_min_std", "up_down", "up_down_dtod",
                  "w_max", "w_min", "w_max_dtod", "w_min_dtod", "slope", "gamma"):
            setattr(od, f, getattr(d, f))
        s.devices[k] = od
        s.gains[k] = g
    s.forward_io = O.default("perfect_io")
    s.backward_io = O.default("perfect_io")
    return O.unitcell(shape[0], shape[1], s, seed)


def test_set_get_forward_backward_match_oracle(restatement):
    """set_weights programs member 0 with w / g0 (clipped) and zeroes the rest;
    the effective weight sum_k g_k W_k drives forward and backward."""
    devs = [const_dev(bound=0.3), const_dev(), const_dev()]
    gains = [2.0, -1.0, 0.5]
    g = cell(devs, gains, xb.UC_ALL_TOGETHER)
    o = oracle_cell(restatement, devs, gains, oracle.UC_ALL_TOGETHER)
    W = np.random.default_rng(1).uniform(-1, 1, (6, 5))
    g.set_weights(W)
    o.set_weights(W)
    assert np.allclose(g.get_weights(), o.get_weights(), atol=1e-6)
    assert np.allclose(g.member(0).get_weights(), o.members[0].get_weights(), atol=1e-6)
    assert not g.member(1).get_weights().any() and not g.member(2).get_weights().any()
    X = np.random.default_rng(2).uniform(-1, 1, (7, 5))
    D = np.random.default_rng(3).uniform(-1, 1, (7, 6))
    Y = g.forward(X)
    G = g.backward(D)
    for b in range(7):
        assert np.allclose(Y[b], o.forward(X[b]), atol=1e-5)
        assert np.allclose(G[b], o.backward(D[b]), atol=1e-5)


def test_single_device_cell_is_the_plain_tile():
    """One device of gain 1: the compound's update stream and member 0 share
    the tile's seed, and the grain is dw_min, so on the GPU the cell reproduces
    the plain tile bit for bit (noise on)."""
    dev = xb.device_preset("reram_sb")
    io = xb.default_io()
    s = xb.UnitCellSettings([dev], [1.0], xb.UC_ALL_TOGETHER, forward_io=io, backward_io=io)
    u = xb.UnitCellTile(32, 48, s, 1234)
    t = xb.AnalogTile(32, 48, xb.TileSettings(device=dev, forward_io=io, backward_io=io), 1234)
    W0 = np.random.default_rng(4).uniform(-0.2, 0.2, (32, 48))
    u.set_weights(W0)
    t.set_weights(W0)
    rng = np.random.default_rng(5)
    for _ in range(3):
        X = rng.uniform(-1, 1, (20, 48)).astype(np.float32)
        D = rng.uniform(-1, 1, (20, 32)).astype(np.float32)
        u.update(X, D, 0.05)
        t.update(X, D, 0.05)
        assert np.array_equal(u.forward(X), t.forward(X))
    assert np.array_equal(u.get_weights(), t.get_weights())


def test_all_together_pair_moves_in_mirror():
    """Gains {+1, -1} on identical noise-free devices: both members fire the
    same trains, member 1 flipped, so W_1 = -W_0 and W_eff = 2 W_0
    (compound.cpp:136-146); each coincidence moves W_eff by the grain 2 dw."""
    dw = 2.0 ** -10
    u = cell([const_dev(dw), const_dev(dw)], [1.0, -1.0], xb.UC_ALL_TOGETHER, shape=(8, 8))
    rng = np.random.default_rng(6)
    X = rng.uniform(-1, 1, (30, 8)).astype(np.float32)
    D = rng.uniform(-1, 1, (30, 8)).astype(np.float32)
    u.update(X, D, 0.02)
    w0, w1 = u.member(0).get_weights(), u.member(1).get_weights()
    assert np.array_equal(w1, -w0)
    assert np.abs(w0).max() > 0
    assert np.array_equal(u.get_weights(), 2 * w0)
    # every change is a whole number of pulses of dw on member 0
    assert np.array_equal(np.round(w0 / dw), w0 / dw)


def test_round_robin_alternates_members():
    """compound.cpp:117-127: sample b goes to member (cursor + b) mod K; zero
    samples neither fire nor advance the cursor; a zero-gain member consumes
    its turn without pulses; the cursor persists across calls."""
    dw = 2.0 ** -8
    devs = [const_dev(dw), const_dev(dw), const_dev(dw)]
    u = cell(devs, [1.0, 0.5, 0.0], xb.UC_ROUND_ROBIN, shape=(4, 3))
    x = np.array([1.0, 1.0, 1.0], np.float32)
    rows = np.eye(4, dtype=np.float32)
    # samples: row0 -> m0, zero sample (skipped), row1 -> m1, row2 -> m2 (gain 0), row3 -> m0
    X = np.stack([x, x, x, x, x])
    D = np.stack([rows[0], np.zeros(4, np.float32), rows[1], rows[2], rows[3]])
    u.update(X, D, 1.0)
    w = [u.member(k).get_weights() for k in range(3)]
    moved = [set(np.nonzero(np.abs(m).sum(axis=1))[0]) for m in w]
    assert moved[0] == {0, 3} and moved[1] == {1} and moved[2] == set()
    u.update(x, rows[2], 1.0)  # cursor continues at member 1
    assert np.abs(u.member(1).get_weights()[2]).sum() > 0


def test_round_robin_expected_update_is_lr_d_x():
    """E[dW_eff] = lr d x^T per sample for any member: the grain |g_k| dw_k
    scales the probabilities so g_k x (#pulses x dw_k) is unbiased."""
    dw = 2.0 ** -12
    u = cell([const_dev(dw), const_dev(dw)], [1.0, -0.5], xb.UC_ROUND_ROBIN, shape=(4, 256))
    x = np.full(256, 0.6, np.float32)
    d = np.array([0.5, -0.25, 0.75, -1.0], np.float32)
    n = 2048
    # lr small enough that no probability clips at 1 (clipping biases the step)
    u.update(np.tile(x, (n, 1)), np.tile(d, (n, 1)), 0.001)
    got = u.get_weights().mean(axis=1) / n
    want = 0.001 * d * 0.6
    assert np.allclose(got, want, rtol=0.03), (got, want)


def test_clone_and_forward_noisy():
    dev = xb.device_preset("reram_sb")
    io = xb.default_io()
    s = xb.UnitCellSettings([dev, dev], [1.0, -0.5], xb.UC_ROUND_ROBIN, forward_io=io,
                            backward_io=io)
    a = xb.UnitCellTile(12, 10, s, 3)
    a.set_weights(np.random.default_rng(7).uniform(-0.2, 0.2, (12, 10)))
    rng = np.random.default_rng(8)
    X = rng.uniform(-1, 1, (9, 10)).astype(np.float32)
    D = rng.uniform(-1, 1, (9, 12)).astype(np.float32)
    a.update(X[:3], D[:3], 0.05)
    c = a.clone()
    a.update(X[3:], D[3:], 0.05)
    c.update(X[3:], D[3:], 0.05)
    assert np.array_equal(a.get_weights(), c.get_weights())
    assert np.array_equal(a.forward(X), c.forward(X))
    p = cell([const_dev(), const_dev()], [1.0, 0.5], xb.UC_ALL_TOGETHER, shape=(8, 64))
    W = np.random.default_rng(9).uniform(-0.3, 0.3, (8, 64))
    p.set_weights(W)
    xv = np.random.default_rng(10).uniform(-1, 1, 64).astype(np.float32)
    Y = p.forward_noisy(np.tile(xv, (4000, 1)), 0.05).astype(np.float64)
    var = 0.05 ** 2 * float(xv.astype(np.float64) @ xv)
    assert np.all(np.abs(Y.mean(axis=0) - W @ xv) < 5 * np.sqrt(var / 4000))
    assert abs(Y.var(axis=0).mean() / var - 1) < 0.06


def test_errors_match_oracle(restatement):
    O = restatement
    cases = []

    def gpu_zero_gain():
        cell([const_dev(), const_dev()], [0.0, 1.0], xb.UC_ALL_TOGETHER).set_weights(
            np.ones((6, 5)))

    def ora_zero_gain():
        oracle_cell(O, [const_dev(), const_dev()], [0.0, 1.0],
                    oracle.UC_ALL_TOGETHER).set_weights(np.ones((6, 5)))

    def gpu_bad_gain():
        cell([const_dev()], [float("inf")], xb.UC_ALL_TOGETHER)

    def ora_bad_gain():
        oracle_cell(O, [const_dev()], [float("inf")], oracle.UC_ALL_TOGETHER)

    def gpu_bad_member():
        bad = const_dev()
        bad.dw_min = -1.0
        cell([const_dev(), bad], [1.0, 1.0], xb.UC_ALL_TOGETHER)

    def ora_bad_member():
        bad = const_dev()
        bad.dw_min = -1.0
        oracle_cell(O, [const_dev(), bad], [1.0, 1.0], oracle.UC_ALL_TOGETHER)

    def gpu_neg_lr():
        cell([const_dev()], [1.0], xb.UC_ROUND_ROBIN).update(np.ones(5), np.ones(6), -0.5)

    def ora_neg_lr():
        oracle_cell(O, [const_dev()], [1.0], oracle.UC_ROUND_ROBIN).update(np.ones(5),
                                                                          np.ones(6), -0.5)

    cases = [(gpu_zero_gain, ora_zero_gain), (gpu_bad_gain, ora_bad_gain),
             (gpu_bad_member, ora_bad_member), (gpu_neg_lr, ora_neg_lr)]
    for g, o in cases:
        with pytest.raises(oracle.OracleError) as eo:
            o()
        with pytest.raises(xb.Error) as eg:
            g()
        assert str(eg.value) == str(eo.value)


def test_eight_members_all_together():
    """The largest cell (XB_MAX_CELL_DEVICES = 8), gains of both signs: every
    member fires the same trains, negative gains flipped, so on identical
    noise-free devices W_k = sign(g_k) W_0 and W_eff = sum |g_k| W_0."""
    dw = 2.0 ** -10
    gains = [1.0, -0.5, 0.25, -2.0, 0.75, -1.0, 1.5, -0.25]
    u = cell([const_dev(dw) for _ in gains], gains, xb.UC_ALL_TOGETHER, shape=(40, 36))
    assert u.n_members() == 8
    rng = np.random.default_rng(16)
    X = rng.uniform(-1, 1, (24, 36)).astype(np.float32)
    D = rng.uniform(-1, 1, (24, 40)).astype(np.float32)
    u.update(X, D, 0.02)
    w0 = u.member(0).get_weights()
    assert np.abs(w0).max() > 0
    for k, gk in enumerate(gains):
        np.testing.assert_array_equal(u.member(k).get_weights(), np.sign(gk) * w0)
    np.testing.assert_allclose(u.get_weights(), sum(abs(g) for g in gains) * w0, rtol=1e-6)
