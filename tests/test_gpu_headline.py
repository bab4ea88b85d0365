"""Parity at the benchmark shapes (BASELINE.json north star: 4096 x 4096 tile,
batch 256), through the C ABI, against the oracle's arithmetic.

* the tcgen05 forward with the default converters (DAC 7 b, ADC 9 b, abs-max;
  output noise off so both sides are deterministic), bound management off
  and on, at 3xTF32 and TF32, vs the fp64 analog_matvec restated per sample
  (proj/src/io.cpp:93-149; the quantizer is pinned to the oracle's);
* the in-kernel bound-management loop (grid barriers, no host round trip)
  vs the host-driven re-issue passes, bit for bit, noise on, one and two
  N slabs;
* the pulsed update of the NS tile (4096^2, B = 256, BL 31, GPU-drawn trains):
  coincidence counts bit-exact for all 16.7 M cells (ConstantStep, dw = 2^-10,
  so W / dw is the signed count), and the reram_sb SoftBounds law on a row
  slice applied by the oracle's apply_pulse_trains with the same trains
  within 1e-5.
"""
import numpy as np
import pytest

import oracle
import paper_2104_02184_b200 as xb
from gpu_helpers import apply_words_to_oracle, close, oracle_settings

pytestmark = pytest.mark.gpu

N = 4096
B = 256


def quantize_np(v, bound, bits):
    """proj/src/io.cpp:42-56 vectorised (round half away from zero)."""
    v = np.asarray(v, dtype=np.float64)
    out = np.clip(v, -bound, bound)
    if bits > 0:
        levels = 2.0 ** bits
        step = 2.0 * bound / levels
        k = (out + bound - 0.5 * step) / step
        k = np.sign(k) * np.floor(np.abs(k) + 0.5)
        k = np.clip(k, 0.0, levels - 1.0)
        out = -bound + (k + 0.5) * step
    return np.where(v == 0.0, 0.0, out)


def test_quantizer_restatement_pinned():
    O = oracle.load("restatement")
    r = np.random.default_rng(0)
    v = np.concatenate([r.uniform(-14, 14, 3000), r.uniform(-1.2, 1.2, 3000), [0.0, 12.0, -12.0]])
    for bound, bits in ((12.0, 9), (1.0, 7), (1.0, 0), (4.0, 3)):
        ref = np.array([O.quantize(x, bound, bits) for x in v])
        assert np.array_equal(quantize_np(v, bound, bits), ref)


def forward_ref(W64, X, io):
    """analog_matvec with sigma_out = 0 per sample, plus the additive
    bound-management rule: the first level m (input / 2^m) whose pre-ADC
    outputs all stay below output_bound, at most bm_max_iter.  Returns y,
    the level per sample and the per-sample margin |max|acc_m| - bound| of
    every level decision taken (a TF32 accumulator may fall on the other
    side of a decision only inside that margin)."""
    alpha = np.abs(X).max(axis=1).astype(np.float64)
    Y = np.zeros((X.shape[0], W64.shape[0]))
    level = np.zeros(X.shape[0], dtype=int)
    margin = np.full(X.shape[0], np.inf)
    pending = np.arange(X.shape[0])
    m = 0
    while len(pending):
        xq = quantize_np(X[pending].astype(np.float64) / (alpha[pending, None] * 2.0 ** m),
                         io.input_bound, io.dac_bits)
        acc = xq @ W64.T
        amax = np.abs(acc).max(axis=1)
        margin[pending] = np.minimum(margin[pending], np.abs(amax - io.output_bound))
        again = (amax >= io.output_bound) & (m < io.bm_max_iter) & bool(io.bound_management)
        done = pending[~again]
        Y[done] = (alpha[done, None] * 2.0 ** m) * quantize_np(acc[~again], io.output_bound,
                                                               io.adc_bits)
        level[done] = m
        pending = pending[again]
        m += 1
    return Y, level, margin, alpha


@pytest.fixture(scope="module")
def headline_inputs():
    r = np.random.default_rng(2024)
    # weights at +-0.3 saturate the 12-unit ADC bound often at 4096 inputs:
    # every sample exercises one or more BM re-issues
    W = r.uniform(-0.3, 0.3, (N, N)).astype(np.float32)
    X = r.uniform(-1, 1, (B, N)).astype(np.float32)
    return W, X


@pytest.mark.parametrize("bm", [False, True])
@pytest.mark.parametrize("prec,lsb_frac,decision_tol", [(xb.MVM_TF32X3, 0.005, 1e-3),
                                                         (xb.MVM_TF32, 0.15, 1e-2)])
def test_forward_converters_headline_shape(headline_inputs, prec, lsb_frac, decision_tol, bm):
    """4096^2 x 256, default converters, BM off/on.  Budget: every output
    within 1 ADC LSB (x alpha 2^m) of the fp64 reference; at most `lsb_frac`
    of them off-grid by that LSB (3xTF32: 0.5 %, TF32: 15 %: a TF32
    accumulator carries ~2^-11 relative error per product, ~2e-3 absolute here
    vs a 0.047 LSB); samples whose BM decision lies within `decision_tol` of
    the bound in fp64 may take the neighbouring level (<= 5 % of samples)."""
    W, X = headline_inputs
    io = xb.default_io()
    io.sigma_out = 0.0
    io.bound_management = xb.BM_ITERATIVE if bm else xb.BM_NONE
    dev = xb.default_device()
    dev.w_max, dev.w_min = 1.0, -1.0
    cfg = xb.TileSettings(device=dev, forward_io=io, backward_io=io, mvm_precision=prec)
    t = xb.AnalogTile(N, N, cfg, 3)
    t.set_weights(W)
    Y = t.forward(X).astype(np.float64)
    ref, level, margin, alpha = forward_ref(W.astype(np.float64), X, io)
    if bm:
        assert level.max() >= 1, "the workload must exercise re-issues"
    lsb = 2 * io.output_bound / 2 ** io.adc_bits * alpha[:, None] * 2.0 ** level[:, None]
    off = np.abs(Y - ref) / lsb
    near = margin < decision_tol
    assert near.mean() <= 0.05
    ok = ~near
    # (1e-4 LSB of slack: alpha 2^m q is rounded to fp32 on the device)
    assert off[ok].max() <= 1.0 + 1e-4, f"max {off[ok].max():.3f} LSB"
    assert (off[ok] > 0.5).mean() <= lsb_frac, f"{(off[ok] > 0.5).mean():.4f} off-grid"


@pytest.mark.parametrize("batch,prec", [(256, xb.MVM_TF32), (100, xb.MVM_TF32),
                                        (300, xb.MVM_TF32), (300, xb.MVM_TF32X3)])
def test_bm_inkernel_loop_equals_host_passes(monkeypatch, headline_inputs, batch, prec):
    """The in-kernel re-issue loop (one launch, grid barriers; at TF32 its
    first re-issue streams the m = 1 slab the idle warps prepared during pass
    0) and the host-enqueued re-issue passes (the row-shard mode: compaction,
    re-issue prep kernel) are bit-identical, with output and weight noise on,
    for one and two N slabs."""
    W, X = headline_inputs
    Xb = np.concatenate([X, X[: batch - B] * 0.5]) if batch > B else X[:batch]
    io = xb.default_io()
    io.sigma_w = 0.01
    io.bound_management = xb.BM_ITERATIVE
    dev = xb.default_device()
    cfg = xb.TileSettings(device=dev, forward_io=io, backward_io=io, mvm_precision=prec)
    out = []
    for host in ("0", "1"):
        monkeypatch.setenv("XB_BM_HOST_PASSES", host)
        t = xb.AnalogTile(N, N, cfg, 17)
        t.set_weights(W)
        out.append((t.forward(Xb), t.forward(Xb)))
    for a, b in zip(out[0], out[1]):
        assert np.array_equal(a, b)


def test_coincidence_counts_ns_shape():
    """Every one of the 4096^2 cells after a GPU-drawn B = 256, BL 31 update:
    W / dw_min equals the signed coincidence count sum_b sum_t
    xbit * dbit * sign exactly (ConstantStep, dw = 2^-10, bounds never hit).
    The reference count comes from the unpacked trains (torch matmul of 0/1
    slot matrices on the GPU, exact in fp32 for these integers)."""
    import torch
    dev = xb.default_device()
    dev.kind, dev.dw_min, dev.w_max, dev.w_min = xb.CONSTANT_STEP, 2.0 ** -10, 10.0, -10.0
    cfg = xb.TileSettings(device=dev)
    t = xb.AnalogTile(N, N, cfg, 5)
    r = np.random.default_rng(9)
    X = r.uniform(-1, 1, (B, N)).astype(np.float32)
    D = r.uniform(-1, 1, (B, N)).astype(np.float32)
    xw, dw, bl = t.generate_trains(X, D, 0.01)
    t.apply_pulse_trains(xw, dw)
    W = t.get_weights()
    cuda = torch.device("cuda")
    xw_t = torch.from_numpy(xw.view(np.int32)).to(cuda)
    dw_t = torch.from_numpy(dw.view(np.int32)).to(cuda)
    sx = torch.where(xw_t < 0, -1.0, 1.0)
    sd = torch.where(dw_t < 0, -1.0, 1.0)
    count = torch.zeros(N, N, device=cuda, dtype=torch.float32)
    for s in range(31):
        xs = ((xw_t >> s) & 1).float() * sx  # [B][N_in]
        ds = ((dw_t >> s) & 1).float() * sd  # [B][N_out]
        count += ds.T @ xs  # direction = sign_d * sign_x (proj/src/pulsed.cpp:96-112)
    assert torch.cuda.is_available()
    expect = count.cpu().numpy().astype(np.float64)
    got = W.astype(np.float64) / dev.dw_min
    assert np.array_equal(got, expect), f"{np.count_nonzero(got != expect)} cells differ"
    assert np.abs(expect).max() > 0


def test_softbounds_update_ns_shape_row_slice():
    """reram_sb law (d2d on, c2c off) on the 4096^2 tile with B = 256 GPU-drawn
    trains; rows [0, 24) are replayed by the oracle's apply_pulse_trains on
    the same realization and weights: within 1e-5 relative."""
    O = oracle.load("restatement")
    dev = xb.device_preset("reram_sb")
    dev.dw_min_std = 0.0
    cfg = xb.TileSettings(device=dev)
    t = xb.AnalogTile(N, N, cfg, 13)
    rows = 24
    o = O.tile(rows, N, oracle_settings(O, cfg), 13)
    up, dn, wmax, wmin = o.get_device()
    upg, dng, wmaxg, wming = t.get_device()
    upg[:rows], dng[:rows], wmaxg[:rows], wming[:rows] = up, dn, wmax, wmin
    t.set_device(upg, dng, wmaxg, wming)
    r = np.random.default_rng(21)
    W0 = r.uniform(-0.1, 0.1, (N, N)).astype(np.float32)
    t.set_weights(W0)
    o.set_weights(t.get_weights()[:rows].astype(np.float64))
    X = r.uniform(-1, 1, (B, N)).astype(np.float32)
    D = r.uniform(-1, 1, (B, N)).astype(np.float32)
    xw, dw, bl = t.generate_trains(X, D, 0.01)
    t.apply_pulse_trains(xw, dw)
    apply_words_to_oracle(o, xw, dw[:, :rows], bl)
    wg, wo = t.get_weights()[:rows], o.get_weights()
    assert close(wg, wo, 1e-5, 0.1).all(), f"max |dw| {np.abs(wg - wo).max():.3e}"
    assert np.abs(wg - W0[:rows]).max() > 0


@pytest.mark.parametrize("prec", [xb.MVM_TF32, xb.MVM_TF32X3])
def test_bm_loop_two_subtile_ctas(monkeypatch, prec):
    """Tiles of >= 8192 rows run the contraction with two 128-row sub-tiles
    per CTA (the cfg5 shape class): the in-kernel re-issue loop there equals
    the host-driven passes bit for bit too (8192 x 1024, B = 256, noise on,
    weights that saturate the ADC bound)."""
    R, C, Bn = 8192, 1024, 256
    r = np.random.default_rng(31)
    W = r.uniform(-0.6, 0.6, (R, C)).astype(np.float32)
    X = r.uniform(-1, 1, (Bn, C)).astype(np.float32)
    io = xb.default_io()
    io.sigma_w = 0.01
    io.bound_management = xb.BM_ITERATIVE
    dev = xb.default_device()
    dev.w_max, dev.w_min = 1.0, -1.0
    cfg = xb.TileSettings(device=dev, forward_io=io, backward_io=io, mvm_precision=prec)
    out = []
    for host in ("0", "1"):
        monkeypatch.setenv("XB_BM_HOST_PASSES", host)
        t = xb.AnalogTile(R, C, cfg, 23)
        t.set_weights(W)
        out.append(t.forward(X))
    np.testing.assert_array_equal(out[0], out[1])
    # the workload re-issues: some sample has outputs beyond alpha * bound,
    # which only a level m >= 1 (scale alpha 2^m) can produce
    alpha = np.abs(X).max(axis=1).astype(np.float64)
    assert (np.abs(out[0]) > io.output_bound * alpha[:, None] * (1 + 1e-6)).any()


@pytest.mark.parametrize("prec", [xb.MVM_TF32, xb.MVM_TF32X3])
def test_bm_loop_backward_equals_host_passes(monkeypatch, headline_inputs, prec):
    """Bound management on the backward (W^T as the MN-major operand): the
    in-kernel re-issue loop equals the host-driven passes bit for bit, noise
    on, at the headline shape."""
    W, X = headline_inputs
    io = xb.default_io()
    io.sigma_w = 0.01
    io.bound_management = xb.BM_ITERATIVE
    dev = xb.default_device()
    cfg = xb.TileSettings(device=dev, forward_io=io, backward_io=io, mvm_precision=prec)
    D = np.random.default_rng(77).uniform(-1, 1, (B, N)).astype(np.float32)
    out = []
    for host in ("0", "1"):
        monkeypatch.setenv("XB_BM_HOST_PASSES", host)
        t = xb.AnalogTile(N, N, cfg, 29)
        t.set_weights(W)
        out.append(t.backward(D))
    np.testing.assert_array_equal(out[0], out[1])
    alpha = np.abs(D).max(axis=1).astype(np.float64)
    assert (np.abs(out[0]) > io.output_bound * alpha[:, None] * (1 + 1e-6)).any()
