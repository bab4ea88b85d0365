"""Pin the plain-C oracle restatement to the reference.

* against tests/golden/golden.npz (generated from the reference build by
  tests/golden/make_golden.py) -- runs everywhere;
* live against oracle/_ref (the reference compiled from its own sources) --
  runs where that library was built.

Bit-exact: the restatement uses the reference's RNG and operation order.
"""
import os

import numpy as np
import pytest

import oracle
import scenarios

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


@pytest.fixture(scope="module")
def restated(restatement):
    return scenarios.run_all(restatement)


def test_impl_names(restatement):
    assert restatement.lib.or_impl_name().decode() == "restatement"


@pytest.mark.parametrize("fn", scenarios.ALL, ids=lambda f: f.__name__)
def test_restatement_matches_golden(golden, restated, fn):
    keys = [k for k in golden.files if k.startswith(fn.__name__ + ".")]
    assert keys, f"no golden arrays for {fn.__name__}"
    for k in keys:
        a, b = restated[k], golden[k]
        assert a.shape == b.shape, k
        assert np.array_equal(a, b), f"{k}: max |diff| {np.max(np.abs(a.astype(float) - b))}"


def test_error_messages_match_golden(golden, restatement):
    msgs = []
    for case in scenarios.error_cases(restatement):
        try:
            case()
            msgs.append("<no error>")
        except oracle.OracleError as e:
            msgs.append(str(e))
    assert msgs == list(golden["errors"])


@pytest.mark.skipif(not oracle.available("reference"), reason="oracle/_ref not built here")
def test_restatement_matches_live_reference(restated):
    ref = scenarios.run_all(oracle.load("reference"))
    for k, v in ref.items():
        assert np.array_equal(restated[k], v), k


# --- the reference's own known-answer tests, re-run through the restatement ---

def test_kat_saturated_trains(restatement):
    """proj/tests/test_pulsed.cpp:66-79: saturated probs -> -31*dw_min exactly."""
    O = restatement
    s = O.default("tile")
    s.device.dw_min, s.device.w_max, s.device.w_min = 0.001, 1.0, -1.0
    s.forward_io = O.default("perfect_io")
    t = O.tile(1, 1, s, 2)
    t.update([1.0], [-1.0], 10.0)
    assert t.get_weights()[0, 0] == pytest.approx(-31 * 0.001, rel=1e-12)


def test_kat_bruteforce_counts(restatement):
    """proj/tests/test_pulsed.cpp:133-158: dW = dw_min * brute-force count."""
    O = restatement
    s = O.default("tile")
    s.device.dw_min, s.device.w_max, s.device.w_min = 0.001, 10.0, -10.0
    t = O.tile(3, 4, s, 6)
    x = np.random.default_rng(7).uniform(-1, 1, 4)
    d = np.random.default_rng(8).uniform(-1, 1, 3)
    up = O.default("update")
    bl, px, pd, sx, sd = O.translate(x, d, 0.02, 0.001, up)
    xb, db = O.generate_trains(bl, px, pd, O.rng(9))
    t.apply_pulse_trains(bl, xb, db, sx, sd)
    w = t.get_weights()
    counts = (db.T.astype(int) @ xb.astype(int))
    np.testing.assert_allclose(w, 0.001 * counts * np.outer(sd, sx), rtol=1e-12, atol=0)


def test_kat_softbounds_closed_form(restatement):
    """acceptance criterion 3 (proj/tests/acceptance_main.cpp:231-249)."""
    import ctypes as C
    O = restatement
    p = O.default("device")
    p.kind, p.dw_min, p.w_max, p.w_min = oracle.SOFT_BOUNDS, 0.01, 0.6, -0.6
    r = O.rng(3001)
    cell = np.zeros(6)
    cp = cell.ctypes.data_as(C.POINTER(C.c_double))
    O.lib.or_realize_cell(p, r.h, cp)
    w, worst = 0.0, 0.0
    for n in range(1, 1001):
        w = O.lib.or_apply_pulse(cp, w, 1, oracle.SOFT_BOUNDS, 0.0, r.h)
        closed = 0.6 - 0.6 * (1 - 0.01 / 0.6) ** n
        worst = max(worst, abs(w - closed))
    assert worst <= 1e-6


def test_kat_drift_factor(restatement):
    """proj/tests/test_inference.cpp:79-97: uniform drift multiplies by (t/t0)^-nu."""
    O = restatement
    s = O.default("tile")
    s.device.w_max, s.device.w_min = 100.0, -100.0
    s.forward_io = O.default("perfect_io")
    t = O.tile(2, 2, s, 11)
    m = O.default("inference")
    m.prog_noise_scale, m.read_noise_scale, m.nu_std, m.t0 = 0.0, 0.0, 0.0, 1.0
    target = np.random.default_rng(12).uniform(-0.5, 0.5, (2, 2))
    w0, nu = t.program(target, m, O.rng(13))
    t.drift_to(w0, nu, 1.0, 100.0)
    np.testing.assert_allclose(t.get_weights(), target * 100.0 ** -0.06, atol=1e-9)
