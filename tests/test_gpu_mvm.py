"""Noisy-MVM parity: the CUDA forward/backward (through the C ABI) vs the oracle.

Noise off: outputs within 1e-5 * max(1, |y|) of the fp64 oracle (the
reference's own tolerance form, proj/tests/test_tile.cpp:263), converters on:
identical grid values except <= 1 ADC LSB on a small fraction (an fp32
accumulator can sit on the other side of an ADC threshold).  Noise on:
moments within stated confidence bounds.
"""
import numpy as np
import pytest

import oracle
import paper_2104_02184_b200 as xb
from gpu_helpers import close, twin

pytestmark = pytest.mark.gpu

# the exact SIMT path and both tcgen05 modes (the samples per call are >= 16,
# so the tensor-core modes really run on tcgen05)
PRECISIONS = [xb.MVM_FP32, xb.MVM_TF32X3, xb.MVM_TF32]
# relative tolerance of the contraction per mode: fp32-level for the SIMT and
# 3xTF32 paths (the reference's 1e-5 form), TF32's 10-bit mantissa otherwise
TOL = {xb.MVM_FP32: 1e-5, xb.MVM_TF32X3: 1e-5, xb.MVM_TF32: 2e-3}


def cfg_io(fwd=None, bwd=None, prec=xb.MVM_FP32, bound=4.0):
    dev = xb.default_device()
    dev.w_max, dev.w_min = bound, -bound
    return xb.TileSettings(device=dev, forward_io=fwd if fwd is not None else xb.io_off(),
                           backward_io=bwd if bwd is not None else xb.io_off(),
                           mvm_precision=prec)


@pytest.mark.parametrize("prec", PRECISIONS)
@pytest.mark.parametrize("shape", [(16, 16), (256, 256), (300, 130)])
@pytest.mark.parametrize("perfect", [True, False])
def test_noise_off_matches_exact_matvec(prec, shape, perfect):
    """proj/tests/test_tile.cpp:225-266 (ideal limit) and io_off paths."""
    io = xb.perfect_io() if perfect else xb.io_off()
    g, o = twin(cfg_io(io, io, prec), *shape, w_scale=0.5)
    nb = 20  # >= 16: the tensor-core modes take the tcgen05 path
    X = np.random.default_rng(61).uniform(-1, 1, (nb, shape[1])).astype(np.float32)
    D = np.random.default_rng(62).uniform(-1, 1, (nb, shape[0])).astype(np.float32)
    Y = g.forward(X)
    G = g.backward(D)
    W = o.get_weights()
    if prec == xb.MVM_TF32:  # relative to the dot-product scale |x| |w_i|
        sy = np.linalg.norm(X, axis=1)[:, None] * np.linalg.norm(W, axis=1)[None, :]
        sg = np.linalg.norm(D, axis=1)[:, None] * np.linalg.norm(W, axis=0)[None, :]
        assert (np.abs(Y - X.astype(np.float64) @ W.T) / sy).max() < TOL[prec]
        assert (np.abs(G - D.astype(np.float64) @ W) / sg).max() < TOL[prec]
        return
    assert close(Y, X.astype(np.float64) @ W.T, TOL[prec], 1.0).all()
    assert close(G, D.astype(np.float64) @ W, TOL[prec], 1.0).all()
    for b in range(nb):
        assert close(Y[b], o.forward(X[b]), TOL[prec], 1.0).all()
        assert close(G[b], o.backward(D[b]), TOL[prec], 1.0).all()


@pytest.mark.parametrize("prec", PRECISIONS)
def test_converters_match_oracle_grid(prec):
    """Default DAC 7 b / ADC 9 b / abs-max, sigma_out = 0: same grid values;
    at most 1 LSB apart on <= 0.5 % of outputs."""
    io = xb.default_io()
    io.sigma_out = 0.0
    g, o = twin(cfg_io(io, io, prec, bound=1.0), 128, 512, w_scale=0.1)
    X = np.random.default_rng(7).uniform(-1, 1, (32, 512)).astype(np.float32)
    Y = g.forward(X)
    ref = np.stack([o.forward(X[b]) for b in range(32)])
    alpha = np.abs(X).max(axis=1, keepdims=True)
    lsb = 2 * 12.0 / 512 * alpha
    diff = np.abs(Y - ref)
    # off-grid budget: 0.5 % for the fp32-level paths; TF32 (~5e-4 absolute
    # error on these dot products vs a 0.047 LSB) up to 5 %
    frac = 0.05 if prec == xb.MVM_TF32 else 0.005
    assert np.all(diff <= lsb * 1.001 + 1e-6)
    assert np.mean(diff > 1e-6 * np.maximum(1, np.abs(ref))) <= frac
    D = np.random.default_rng(8).uniform(-1, 1, (32, 128)).astype(np.float32)
    G = g.backward(D)
    refg = np.stack([o.backward(D[b]) for b in range(32)])
    lsbg = 2 * 12.0 / 512 * np.abs(D).max(axis=1, keepdims=True)
    assert np.all(np.abs(G - refg) <= lsbg * 1.001 + 1e-6)


def test_outputs_on_adc_grid():
    """proj/tests/test_tile.cpp:406-421."""
    io = xb.io_off()
    io.adc_bits, io.output_bound = 4, 2.0
    g = xb.AnalogTile(3, 3, cfg_io(io), 19)
    g.set_weights(np.random.default_rng(95).uniform(-0.4, 0.4, (3, 3)))
    y = g.forward(np.random.default_rng(96).uniform(-0.9, 0.9, 3))
    step = 2 * 2.0 / 16
    k = (y + 2.0 - 0.5 * step) / step
    assert np.all(np.abs(k - np.round(k)) < 1e-5)


def test_zero_input():
    """proj/tests/test_tile.cpp:66-82 and io.cpp:107-115."""
    io = xb.default_io()
    io.sigma_inp, io.sigma_w, io.sigma_out = 0.1, 0.2, 0.0
    g = xb.AnalogTile(3, 4, cfg_io(io), 1)
    g.set_weights(np.random.default_rng(9).uniform(-0.5, 0.5, (3, 4)))
    assert np.all(g.forward(np.zeros(4)) == 0.0)
    io.sigma_out = 0.1
    g2 = xb.AnalogTile(200, 4, cfg_io(io), 1)
    y = g2.forward(np.zeros((50, 4)))
    step = 2 * 12.0 / 512
    assert abs(y.std() - 0.1) < 0.01  # noise-only path, then the ADC
    k = (y + 12.0 - 0.5 * step) / step
    assert np.all(np.abs(k - np.round(k)) < 1e-3)


def test_forward_unbiased_and_noise_variance():
    """test_tile.cpp:145-174: all noise on, converters off: mean = W x, and
    var = sigma_out^2 + sigma_w^2 ||x~||^2 + sigma_inp^2 ||w_i||^2."""
    io = xb.io_off()
    io.input_bound = io.output_bound = 1e6
    io.sigma_inp, io.sigma_out, io.sigma_w = 0.03, 0.05, 0.02
    io.noise_management = xb.NM_ABS_MAX
    g = xb.AnalogTile(3, 4, cfg_io(io), 6)
    W = np.random.default_rng(21).uniform(-0.4, 0.4, (3, 4)).astype(np.float32)
    g.set_weights(W)
    x = np.random.default_rng(22).uniform(-0.8, 0.8, 4).astype(np.float32)
    n = 60000
    Y = g.forward(np.tile(x, (n, 1))).astype(np.float64)
    exact = W.astype(np.float64) @ x
    se = Y.std(axis=0) / np.sqrt(n)
    assert np.all(np.abs(Y.mean(axis=0) - exact) < 4 * se)
    alpha = np.abs(x).max()
    xn = x / alpha
    var = alpha ** 2 * (0.05 ** 2 + 0.02 ** 2 * (xn @ xn + 4 * 0.03 ** 2)
                        + 0.03 ** 2 * (W.astype(np.float64) ** 2).sum(axis=1))
    ratio = Y.var(axis=0) / var
    assert np.all(np.abs(ratio - 1) < 0.05), ratio


def test_abs_max_scale_invariance():
    """proj/tests/test_tile.cpp:176-198: same seed -> same noise draws."""
    io = xb.io_off()
    io.sigma_inp, io.sigma_out, io.noise_management = 0.02, 0.05, xb.NM_ABS_MAX
    a = xb.AnalogTile(3, 4, cfg_io(io), 77)
    b = xb.AnalogTile(3, 4, cfg_io(io), 77)
    W = np.random.default_rng(31).uniform(-0.4, 0.4, (3, 4))
    a.set_weights(W)
    b.set_weights(W)
    x = np.random.default_rng(32).uniform(-0.6, 0.6, 4).astype(np.float32)
    c = np.float32(4.0)  # power of two keeps x / alpha bit-identical in fp32
    np.testing.assert_allclose(b.forward(c * x), c * a.forward(x), rtol=1e-6)


def test_determinism_same_seed():
    """proj/tests/test_tile.cpp:200-223."""
    dev = xb.default_device()
    dev.dw_min_dtod, dev.dw_min_std = 0.3, 0.3
    s = xb.TileSettings(device=dev)
    a = xb.AnalogTile(4, 4, s, 123)
    b = xb.AnalogTile(4, 4, s, 123)
    W = np.random.default_rng(41).uniform(-0.3, 0.3, (4, 4))
    a.set_weights(W)
    b.set_weights(W)
    x = np.random.default_rng(42).uniform(-0.9, 0.9, 4)
    d = np.random.default_rng(43).uniform(-0.5, 0.5, 4)
    for _ in range(5):
        np.testing.assert_array_equal(a.forward(x), b.forward(x))
        a.update(x, d, 0.01)
        b.update(x, d, 0.01)
    np.testing.assert_array_equal(a.get_weights(), b.get_weights())


def test_read_noise_never_lands_in_the_array():
    """proj/tests/test_tile.cpp:268-291."""
    io = xb.default_io()
    io.sigma_out, io.sigma_w = 0.1, 0.1
    g = xb.AnalogTile(2, 2, cfg_io(io, bound=1.0), 11)
    g.set_weights([[0.5, -0.25], [10.0, 0.0]])
    got = g.get_weights()
    np.testing.assert_array_equal(got, np.array([[0.5, -0.25], [1.0, 0.0]], np.float32))
    g.forward(np.tile([0.3, 0.4], (50, 1)))
    np.testing.assert_array_equal(g.get_weights(), got)


def test_backward_is_forward_of_transpose():
    """proj/tests/test_tile.cpp:200-223 (ideal backward == forward on W^T)."""
    s = cfg_io(xb.perfect_io(), xb.perfect_io())
    W = np.random.default_rng(51).uniform(-0.4, 0.4, (5, 7))
    a = xb.AnalogTile(5, 7, s, 8)
    a.set_weights(W)
    t = xb.AnalogTile(7, 5, s, 9)
    t.set_weights(W.T)
    d = np.random.default_rng(52).uniform(-1, 1, 5)
    np.testing.assert_allclose(a.backward(d), t.forward(d), rtol=1e-6, atol=1e-7)


def test_forward_noisy_read_noise():
    """forward_noisy == forward with sigma_w = hypot(sigma_w, extra) (io.cpp:74-91)."""
    s = cfg_io(xb.perfect_io(), xb.perfect_io())
    g = xb.AnalogTile(64, 256, s, 3)
    W = np.random.default_rng(1).uniform(-0.3, 0.3, (64, 256)).astype(np.float32)
    g.set_weights(W)
    x = np.random.default_rng(2).uniform(-1, 1, 256).astype(np.float32)
    Y = g.forward_noisy(np.tile(x, (4000, 1)), 0.05).astype(np.float64)
    exact = W.astype(np.float64) @ x
    var = 0.05 ** 2 * float(x.astype(np.float64) @ x)
    assert np.all(np.abs(Y.mean(axis=0) - exact) < 5 * np.sqrt(var / 4000))
    assert abs(Y.var(axis=0).mean() / var - 1) < 0.05


@pytest.mark.parametrize("shape,B", [((256, 256), 16), ((300, 520), 37), ((512, 4096), 256),
                                     ((128, 64), 300), ((8320, 200), 40)])
def test_tcgen05_tf32_forward(shape, B):
    """The tcgen05 kind::tf32 contraction (TMA + TMEM, split-K) against the fp32
    SIMT path on the same weights: TF32 keeps 10 mantissa bits, so outputs
    agree to ~1e-3 of max(1, |y|) and must NOT be bit-identical (proof that the
    tensor-core path ran)."""
    d_out, d_in = shape
    io = xb.perfect_io()
    W = np.random.default_rng(3).uniform(-0.5, 0.5, shape).astype(np.float32)
    X = np.random.default_rng(4).uniform(-1, 1, (B, d_in)).astype(np.float32)
    ref = X.astype(np.float64) @ W.T.astype(np.float64)
    out = {}
    for prec in (xb.MVM_FP32, xb.MVM_TF32, xb.MVM_TF32X3):
        t = xb.AnalogTile(d_out, d_in, cfg_io(io, io, prec), 5)
        t.set_weights(W)
        out[prec] = t.forward(X).astype(np.float64)
    # error relative to the dot-product scale ||w_i|| ||x_b|| (Cauchy-Schwarz bound of |y|):
    # fp32 accumulation over K = 4096 terms cannot meet 1e-5 of max(1, |y|) near y = 0
    scale = np.linalg.norm(X.astype(np.float64), axis=1)[:, None] * \
        np.linalg.norm(W.astype(np.float64), axis=1)[None, :]
    err32 = np.abs(out[xb.MVM_FP32] - ref) / scale
    errtf = np.abs(out[xb.MVM_TF32] - ref) / scale
    errx3 = np.abs(out[xb.MVM_TF32X3] - ref) / scale
    assert err32.max() < 1e-5, err32.max()
    assert errtf.max() < 2e-3, errtf.max()
    # 3xTF32 (hi*hi + hi*lo + lo*hi on tcgen05) recovers fp32-level products
    assert errx3.max() < 1e-5, errx3.max()
    assert not np.array_equal(out[xb.MVM_FP32], out[xb.MVM_TF32])
    assert not np.array_equal(out[xb.MVM_FP32], out[xb.MVM_TF32X3])


def test_tcgen05_noisy_forward_statistics():
    """Default IO (DAC 7 b, ADC 9 b, sigma_out 0.06, abs-max) on the tensor-core
    path: mean over repeats matches the fp64 noisy-free reference within the
    ADC/noise budget."""
    io = xb.default_io()
    W = np.random.default_rng(5).uniform(-0.1, 0.1, (256, 1024)).astype(np.float32)
    x = np.random.default_rng(6).uniform(-1, 1, 1024).astype(np.float32)
    t = xb.AnalogTile(256, 1024, cfg_io(io, io, xb.MVM_TF32, bound=1.0), 8)
    t.set_weights(W)
    Y = t.forward(np.tile(x, (512, 1))).astype(np.float64)
    alpha = np.abs(x).max()
    xq = np.array([O_quant(v / alpha) for v in x])
    exact = alpha * (W.astype(np.float64) @ xq)
    se = Y.std(axis=0) / np.sqrt(512)
    assert np.mean(np.abs(Y.mean(axis=0) - exact) < 5 * se + 2e-3) > 0.99
    assert abs(Y.std(axis=0).mean() / (alpha * np.sqrt(0.06 ** 2 + (24 / 512) ** 2 / 12)) - 1) < 0.1


def O_quant(v, bound=1.0, bits=7):
    return oracle.load("restatement").quantize(v, bound, bits)


def bm_forward_ref(W, x, io, O):
    """Restatement of the additive bound-management rule (no reference symbol;
    DESIGN.md): re-issue with the input halved until no pre-ADC output reaches
    output_bound or bm_max_iter is hit; y = alpha 2^m ADC(acc_m)."""
    alpha = np.abs(x).max()
    if alpha == 0:
        return np.zeros(W.shape[0])
    if io.noise_management != xb.NM_ABS_MAX:
        alpha = 1.0
    m = 0
    while True:
        xt = np.array([O.quantize(v / (alpha * 2.0 ** m), io.input_bound, io.dac_bits) for v in x])
        acc = W.astype(np.float64) @ xt
        if np.abs(acc).max() >= io.output_bound and m < io.bm_max_iter:
            m += 1
            continue
        return alpha * 2.0 ** m * np.array([O.quantize(a, io.output_bound, io.adc_bits)
                                            for a in acc])


@pytest.mark.parametrize("prec", [xb.MVM_FP32, xb.MVM_TF32])
def test_bound_management_reissue(prec):
    """Saturating samples are re-issued at half input scale until the ADC no
    longer clips; non-saturating samples are untouched."""
    O = oracle.load("restatement")
    io = xb.default_io()
    io.sigma_out = 0.0
    io.bound_management, io.bm_max_iter = xb.BM_ITERATIVE, 5
    W = np.full((24, 64), 0.9, np.float32)
    W[::2] *= -0.25
    X = np.random.default_rng(3).uniform(0.2, 1.0, (20, 64)).astype(np.float32)
    X[::3] *= 0.05  # tiny samples still saturate: abs-max rescales them to full range
    X[1::4] = np.random.default_rng(4).uniform(-1, 1, (len(X[1::4]), 64))  # cancellations
    t = xb.AnalogTile(24, 64, cfg_io(io, io, prec, bound=1.0), 2)
    t.set_weights(W)
    Y = t.forward(X)
    for b in range(X.shape[0]):
        ref = bm_forward_ref(W, X[b].astype(np.float64), io, O)
        lsb = 2 * 12.0 / 512 * np.abs(X[b]).max() * 2 ** 5
        assert np.all(np.abs(Y[b] - ref) <= lsb), (b, Y[b][:4], ref[:4])
    # without BM the same tile clips at alpha * 12
    io.bound_management = xb.BM_NONE
    t2 = xb.AnalogTile(24, 64, cfg_io(io, io, prec, bound=1.0), 2)
    t2.set_weights(W)
    Y2 = t2.forward(X)
    assert np.abs(Y2).max() <= 12.0 * np.abs(X).max() + 1e-5
    assert np.abs(Y).max() > 20.0


@pytest.mark.parametrize("shape,B", [((256, 256), 16), ((520, 300), 37), ((4096, 512), 256),
                                     ((45, 37), 20), ((130, 77), 300), ((96, 8320), 24)])
def test_tcgen05_tf32_backward(shape, B):
    """Backward contraction W^T d on tcgen05 with the MN-major A operand
    (four 32x32 TMA boxes per stage) against the fp32 SIMT path."""
    d_out, d_in = shape
    io = xb.perfect_io()
    W = np.random.default_rng(13).uniform(-0.5, 0.5, shape).astype(np.float32)
    D = np.random.default_rng(14).uniform(-1, 1, (B, d_out)).astype(np.float32)
    ref = D.astype(np.float64) @ W.astype(np.float64)
    out = {}
    for prec in (xb.MVM_FP32, xb.MVM_TF32, xb.MVM_TF32X3):
        t = xb.AnalogTile(d_out, d_in, cfg_io(io, io, prec), 5)
        t.set_weights(W)
        out[prec] = t.backward(D).astype(np.float64)
    scale = np.linalg.norm(D.astype(np.float64), axis=1)[:, None] * \
        np.linalg.norm(W.astype(np.float64), axis=0)[None, :]
    assert (np.abs(out[xb.MVM_FP32] - ref) / scale).max() < 1e-5
    assert (np.abs(out[xb.MVM_TF32] - ref) / scale).max() < 2e-3
    assert (np.abs(out[xb.MVM_TF32X3] - ref) / scale).max() < 1e-5
    if B >= 16:
        assert not np.array_equal(out[xb.MVM_FP32], out[xb.MVM_TF32])
        assert not np.array_equal(out[xb.MVM_FP32], out[xb.MVM_TF32X3])


def test_tcgen05_forward_odd_widths():
    """Columns not a multiple of 4 (padded x~ stride for TMA) and rows not a
    multiple of 128."""
    io = xb.perfect_io()
    W = np.random.default_rng(15).uniform(-0.5, 0.5, (77, 45)).astype(np.float32)
    X = np.random.default_rng(16).uniform(-1, 1, (40, 45)).astype(np.float32)
    t = xb.AnalogTile(77, 45, cfg_io(io, io, xb.MVM_TF32), 5)
    t.set_weights(W)
    Y = t.forward(X).astype(np.float64)
    ref = X.astype(np.float64) @ W.T.astype(np.float64)
    scale = np.linalg.norm(X, axis=1)[:, None] * np.linalg.norm(W, axis=1)[None, :]
    assert (np.abs(Y - ref) / scale).max() < 2e-3


@pytest.mark.parametrize("prec", [xb.MVM_TF32, xb.MVM_TF32X3])
@pytest.mark.parametrize("shape,B,bm", [((4096, 1024), 256, True), ((520, 300), 37, False),
                                        ((8320, 200), 40, True), ((300, 4096), 300, False),
                                        ((512, 256), 300, True)])
def test_fused_epilogue_matches_unfused(monkeypatch, prec, shape, B, bm):
    """The cluster-fused output stage (K-splits reduced through distributed
    shared memory inside the tcgen05 kernel) and the split-K partials +
    epilogue kernel path produce bit-identical outputs, noise and BM included."""
    d_out, d_in = shape
    io = xb.default_io()
    io.bound_management = xb.BM_ITERATIVE if bm else xb.BM_NONE
    io.sigma_w = 0.02
    W = np.random.default_rng(21).uniform(-0.3, 0.3, shape).astype(np.float32)
    X = np.random.default_rng(22).uniform(-1, 1, (B, d_in)).astype(np.float32)
    D = np.random.default_rng(23).uniform(-1, 1, (B, d_out)).astype(np.float32)
    out = []
    for unfused in ("0", "1"):
        monkeypatch.setenv("XB_MVM_UNFUSED", unfused)
        t = xb.AnalogTile(d_out, d_in, cfg_io(io, io, prec), 31)
        t.set_weights(W)
        out.append((t.forward(X), t.backward(D), t.forward(X)))
    for a, b in zip(out[0], out[1]):
        assert np.array_equal(a, b)


def test_forward_into_caller_buffer():
    """forward(x, out=Y) writes into the caller's (e.g. pinned) float32 buffer
    and returns it; shape/dtype mismatches raise."""
    t = xb.AnalogTile(64, 32, cfg_io(xb.perfect_io(), xb.perfect_io(), xb.MVM_FP32), 3)
    W = np.random.default_rng(1).uniform(-0.5, 0.5, (64, 32)).astype(np.float32)
    t.set_weights(W)
    X = np.random.default_rng(2).uniform(-1, 1, (5, 32)).astype(np.float32)
    Y = np.empty((5, 64), np.float32)
    assert t.forward(X, out=Y) is Y
    assert np.array_equal(Y, t.forward(X))
    with pytest.raises(xb.Error, match="out:"):
        t.forward(X, out=np.empty((5, 63), np.float32))
    with pytest.raises(xb.Error, match="out:"):
        t.forward(X, out=np.empty((5, 64), np.float64))


@pytest.mark.parametrize("prec", PRECISIONS)
def test_dac_exact_including_ties(prec):
    """The DAC (fp32 fast path with an fp64 fallback near grid ties) equals the
    reference quantizer bit for bit (proj/src/io.cpp:42-56,122-130): an
    identity tile, ADC off, abs-max on, y = alpha * Q_dac(x / alpha); inputs
    include values one fp32 ulp either side of every grid threshold."""
    O = oracle.load("restatement")
    n = 256
    io = xb.io_off()
    io.dac_bits, io.input_bound, io.noise_management = 7, 1.0, xb.NM_ABS_MAX
    t = xb.AnalogTile(n, n, cfg_io(io, io, prec, bound=2.0), 3)
    t.set_weights(np.eye(n, dtype=np.float32))
    r = np.random.default_rng(5)
    B = 32
    X = r.uniform(-1, 1, (B, n)).astype(np.float32)
    X[:, 0] = 1.0  # alpha = 1: thresholds of the 7-bit grid at (j / 64) - 1
    thr = (np.arange(1, 128) / 64.0 - 1.0).astype(np.float32)
    X[1:, 1:128] = thr[None, :]
    X[1:8, 1:128] = np.nextafter(thr, np.float32(2.0))[None, :]
    X[8:16, 1:128] = np.nextafter(thr, np.float32(-2.0))[None, :]
    X[16:, 1:64] = 0.0
    Y = t.forward(X).astype(np.float64)
    alpha = np.abs(X).max(axis=1).astype(np.float64)
    ref = np.array([[alpha[b] * O.quantize(float(X[b, j]) / alpha[b], 1.0, 7) for j in range(n)]
                    for b in range(B)]).astype(np.float32)
    if prec == xb.MVM_TF32:
        # the identity contraction on TF32 keeps the 7-bit grid values exactly
        assert np.array_equal(Y.astype(np.float32), ref)
    else:
        assert np.array_equal(Y.astype(np.float32), ref)


@pytest.mark.parametrize("B", [1, 3, 8, 15])
@pytest.mark.parametrize("shape", [(4096, 4096), (77, 45), (300, 130), (1, 513), (513, 1)])
def test_small_batch_gemv_matches_fp64(B, shape):
    """Batches of <= 15 samples (every per-sample reference call) take the
    streaming GEMV kernels (forward: warp per 2 rows; backward: row splits
    summed in order): fp32-exact to 1e-5 of max(1, |y|) against fp64, every
    precision mode (the tensor cores serve B >= 16 only), odd widths."""
    d_out, d_in = shape
    W = np.random.default_rng(41).uniform(-0.5, 0.5, shape).astype(np.float32)
    X = np.random.default_rng(42).uniform(-1, 1, (B, d_in)).astype(np.float32)
    D = np.random.default_rng(43).uniform(-1, 1, (B, d_out)).astype(np.float32)
    for prec in PRECISIONS:
        t = xb.AnalogTile(d_out, d_in, cfg_io(xb.perfect_io(), xb.perfect_io(), prec), 5)
        t.set_weights(W)
        Y = t.forward(X)
        G = t.backward(D)
        assert close(Y, X.astype(np.float64) @ W.T.astype(np.float64), 1e-5, 1.0).all()
        assert close(G, D.astype(np.float64) @ W.astype(np.float64), 1e-5, 1.0).all()


@pytest.mark.parametrize("B", [1, 5, 15])
@pytest.mark.parametrize("shape", [(4096, 4096), (260, 77)])
def test_fused_small_batch_forward_equals_staged_path(monkeypatch, B, shape):
    """Small batches run prep + contraction + output stage as ONE kernel (the
    DAC on the fly, gemv_fused_fwd_kernel); with the default converters and
    output noise it equals the staged path (prep kernel, GEMV, epilogue
    kernel; forced by XB_MVM_UNFUSED) bit for bit -- same DAC grid, same
    contraction order, same noise words -- including an all-zero sample."""
    d_out, d_in = shape
    io = xb.default_io()  # DAC 7 b, ADC 9 b, sigma_out 0.06, abs-max
    W = np.random.default_rng(51).uniform(-0.4, 0.4, shape).astype(np.float32)
    X = np.random.default_rng(52).uniform(-1, 1, (B, d_in)).astype(np.float32)
    X[0, : d_in // 3] = np.linspace(-1, 1, d_in // 3) * 0.5  # exact DAC thresholds
    if B > 1:
        X[1] = 0.0
    out = []
    for unfused in ("0", "1"):
        monkeypatch.setenv("XB_MVM_UNFUSED", unfused)
        t = xb.AnalogTile(d_out, d_in, cfg_io(io, io, xb.MVM_FP32), 77)
        t.set_weights(W)
        out.append((t.forward(X), t.forward(X)))
    for a, b in zip(out[0], out[1]):
        np.testing.assert_array_equal(a, b)
    assert not np.array_equal(out[0][0], out[0][1])  # fresh noise per call


def test_fused_small_batch_forward_weight_noise_equals_staged(monkeypatch):
    """With weight noise (sigma_w ||x~|| zeta) the fused kernel's ||x~|| is the
    prep kernel's to the bit (same per-thread partials, same reduction order)."""
    io = xb.default_io()
    io.sigma_w = 0.05
    W = np.random.default_rng(61).uniform(-0.4, 0.4, (512, 5000)).astype(np.float32)
    X = np.random.default_rng(62).uniform(-1, 1, (3, 5000)).astype(np.float32)
    out = []
    for unfused in ("0", "1"):
        monkeypatch.setenv("XB_MVM_UNFUSED", unfused)
        t = xb.AnalogTile(512, 5000, cfg_io(io, io, xb.MVM_FP32), 78)
        t.set_weights(W)
        out.append(t.forward(X))
    np.testing.assert_array_equal(out[0], out[1])
