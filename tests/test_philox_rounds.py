"""The c2c factors of the pulse kernel draw from Philox4x32 with 7 rounds
(csrc/xb_update.cu, XB_C2C_ROUNDS; Salmon et al., SC'11: Philox4x32 passes
TestU01 BigCrush from 7 rounds).  This CPU test restates Philox4x32-R in
numpy and checks the 7-round stream on the kernel's exact counter pattern --
(3 m + {0,1,2}, column j, row i, call) per cell, neighbouring cells and
words -- for uniformity (every bit, byte and 16-bit radius field), for
independence of neighbouring counters, and against the 10-round stream on
the same statistics.  (The GPU tests then pin the resulting per-pulse
weight-change distribution for all four device laws.)"""
import numpy as np
import pytest

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK = np.uint64(0xFFFFFFFF)


def philox(c0, c1, c2, c3, k0, k1, rounds):
    """Philox4x32-R (xb_common.cuh: philox_round), vectorised over counters."""
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint64) for c in (c0, c1, c2, c3))
    for r in range(rounds):
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK
        kk0 = np.uint64((k0 + r * W0) & 0xFFFFFFFF)
        kk1 = np.uint64((k1 + r * W1) & 0xFFFFFFFF)
        c0, c1, c2, c3 = hi1 ^ c1 ^ kk0, lo1, hi0 ^ c3 ^ kk1, lo0
    return [c.astype(np.uint32) for c in (c0, c1, c2, c3)]


def test_philox10_known_answer():
    """Random123's published known-answer vector for Philox4x32-10
    (kat_vectors: counter = key = 0)."""
    out = philox(0, 0, 0, 0, 0, 0, 10)
    assert [int(x) for x in out] == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]


def kernel_stream(rounds, rows=128, cols=128, groups=12, call=3):
    """The words the pulse kernel draws for `groups` Philox calls of every
    cell (i, j) of a rows x cols patch (counter layout of word32())."""
    g, j, i = np.meshgrid(np.arange(groups), np.arange(cols), np.arange(rows), indexing="ij")
    k0, k1 = 0x1234ABCD, 0x0BADF00D
    return np.stack(philox(g.ravel(), j.ravel(), i.ravel(), np.full(g.size, call), k0, k1,
                           rounds)), g.shape


@pytest.mark.parametrize("rounds", [7, 10])
def test_c2c_stream_uniform_and_independent(rounds):
    words, shape = kernel_stream(rounds)
    w = words.ravel()
    n = w.size  # 786 432 words
    # every bit position: frequency 1/2 within 5 sigma
    bits = ((w[:, None] >> np.arange(32, dtype=np.uint32)) & 1).mean(axis=0)
    assert np.all(np.abs(bits - 0.5) < 5 * 0.5 / np.sqrt(n))
    # byte values: chi-square over 256 bins, each of the 4 bytes
    for s in (0, 8, 16, 24):
        cnt = np.bincount((w >> np.uint32(s)) & 0xFF, minlength=256)
        chi2 = ((cnt - n / 256) ** 2 / (n / 256)).sum()
        assert chi2 < 255 + 6 * np.sqrt(2 * 255)
    # the 16-bit radius fields (upper halves) in 256 bins
    cnt = np.bincount((w >> np.uint32(24)), minlength=256)
    assert ((cnt - n / 256) ** 2 / (n / 256)).sum() < 255 + 6 * np.sqrt(2 * 255)
    # neighbouring counters (next column j, next row i, next call group g):
    # Pearson correlation of the uniforms ~ 0
    u = (words[0].astype(np.float64) / 2 ** 32).reshape(shape)
    for a, b in ((u[:, :-1], u[:, 1:]), (u[:, :, :-1], u[:, :, 1:]), (u[:-1], u[1:])):
        r = np.corrcoef(a.ravel(), b.ravel())[0, 1]
        assert abs(r) < 5 / np.sqrt(a.size)
    # the four output words of one call
    for p in range(1, 4):
        r = np.corrcoef(words[0].astype(np.float64), words[p].astype(np.float64))[0, 1]
        assert abs(r) < 5 / np.sqrt(words.shape[1])


def test_seven_and_ten_rounds_agree_in_distribution():
    """Two-sample KS of the 7- and 10-round uniforms on the kernel pattern."""
    from scipy.stats import ks_2samp
    a = kernel_stream(7)[0][1].astype(np.float64)
    b = kernel_stream(10)[0][1].astype(np.float64)
    assert ks_2samp(a, b).pvalue > 1e-3
