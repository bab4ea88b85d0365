"""Row sharding on one GPU: two shard handles of one logical tile reproduce
the unsharded tile (Philox draws are keyed on global rows).  Here the
collective (max over shards of max|d|, sum of backward partials) is done by
hand between the split-phase entries; tests/test_gpu_comm.py runs the same
through the library's communicators (xb_comm)."""
import numpy as np
import pytest
import torch

import paper_2104_02184_b200 as xb

pytestmark = pytest.mark.gpu


def cfg(prec=xb.MVM_FP32):
    return xb.TileSettings(device=xb.device_preset("reram_sb"), mvm_precision=prec)


@pytest.mark.parametrize("R,C,B", [(96, 80, 40), (256, 130, 300)])
def test_sharded_update_is_bit_identical(R, C, B):
    full = xb.AnalogTile(R, C, cfg(), 77)
    h = R // 2 + 3
    shards = [xb.AnalogTile(R, C, cfg(), 77, shard=(0, h)),
              xb.AnalogTile(R, C, cfg(), 77, shard=(h, R))]
    W = np.random.default_rng(1).uniform(-0.2, 0.2, (R, C)).astype(np.float32)
    full.set_weights(W)
    shards[0].set_weights(W[:h])
    shards[1].set_weights(W[h:])
    # identical per-cell realizations (global-index Philox)
    for a, b in zip(full.get_device(), [np.vstack(x) for x in zip(*[s.get_device() for s in shards])]):
        np.testing.assert_array_equal(a, b)
    g = torch.Generator(device="cuda").manual_seed(3)
    X = torch.rand(B, C, device="cuda", generator=g) * 2 - 1
    D = torch.rand(B, R, device="cuda", generator=g) * 2 - 1
    full.update_dev(X, D, 0.01)
    full.synchronize()
    parts = [D[:, :h].contiguous(), D[:, h:].contiguous()]
    amax = torch.maximum(shards[0].rows_amax(parts[0]), shards[1].rows_amax(parts[1]))
    torch.cuda.synchronize()
    for s, p in zip(shards, parts):
        s.update_dev(X, p, 0.01, amax_d=amax)
        s.synchronize()
    np.testing.assert_array_equal(full.get_weights(),
                                  np.vstack([s.get_weights() for s in shards]))


def test_sharded_forward_is_bit_identical():
    R, C, B = 200, 96, 33
    full = xb.AnalogTile(R, C, cfg(), 5)
    shards = [xb.AnalogTile(R, C, cfg(), 5, shard=(0, 120)),
              xb.AnalogTile(R, C, cfg(), 5, shard=(120, R))]
    W = np.random.default_rng(2).uniform(-0.3, 0.3, (R, C)).astype(np.float32)
    full.set_weights(W)
    shards[0].set_weights(W[:120])
    shards[1].set_weights(W[120:])
    X = np.random.default_rng(4).uniform(-1, 1, (B, C)).astype(np.float32)
    Yf = full.forward(X)
    Ys = np.hstack([s.forward(X) for s in shards])
    np.testing.assert_array_equal(Yf, Ys)


def test_sharded_backward_matches_within_one_lsb():
    """Partial column sums per shard + sum + finish == the unsharded backward
    up to fp32 summation order (at most one ADC step)."""
    R, C, B = 160, 72, 24
    full = xb.AnalogTile(R, C, cfg(), 9)
    shards = [xb.AnalogTile(R, C, cfg(), 9, shard=(0, 64)),
              xb.AnalogTile(R, C, cfg(), 9, shard=(64, R))]
    W = np.random.default_rng(5).uniform(-0.3, 0.3, (R, C)).astype(np.float32)
    full.set_weights(W)
    shards[0].set_weights(W[:64])
    shards[1].set_weights(W[64:])
    g = torch.Generator(device="cuda").manual_seed(6)
    D = torch.rand(B, R, device="cuda", generator=g) * 2 - 1
    Gf = torch.empty(B, C, device="cuda")
    full.backward_dev(D, Gf)
    full.synchronize()
    parts = [D[:, :64].contiguous(), D[:, 64:].contiguous()]
    amax = torch.maximum(shards[0].rows_amax(parts[0]), shards[1].rows_amax(parts[1]))
    torch.cuda.synchronize()
    P = [s.backward_partial_dev(p, amax) for s, p in zip(shards, parts)]
    for s in shards:
        s.synchronize()
    Psum = P[0] + P[1]
    torch.cuda.synchronize()
    Gs = torch.empty(B, C, device="cuda")
    shards[0].backward_finish_dev(Psum, amax, Gs)
    shards[0].synchronize()
    lsb = (2 * 12.0 / 512) * amax.cpu().numpy()[:, None]
    diff = np.abs(Gf.cpu().numpy() - Gs.cpu().numpy())
    assert np.all(diff <= lsb * 1.001 + 1e-6)
    assert np.mean(diff > 1e-6) < 0.02


@pytest.mark.parametrize("prec", [xb.MVM_TF32, xb.MVM_FP32])
def test_chunked_backward_equals_one_shot(prec):
    """The split-phase backward entries in sample chunks -- partials issued
    ahead of their finishes (FIFO), as the sharded backward does to overlap
    each chunk's reduction with the next contraction -- draw the same noise as
    one call over the batch: G is bit-identical, and the tile's backward
    counter ends in the same place (a following backward agrees too)."""
    R, C, B = 192, 160, 256
    bio = xb.default_io()
    bio.bound_management = xb.BM_NONE
    s = xb.TileSettings(device=xb.device_preset("reram_sb"), backward_io=bio, mvm_precision=prec)
    W = np.random.default_rng(8).uniform(-0.3, 0.3, (R, C)).astype(np.float32)
    stream = torch.cuda.current_stream()

    def run(t, D, G, chunks):
        amax = t.rows_amax(D)
        edges = [B * k // chunks for k in range(chunks + 1)]
        parts = [(b0, b1, t.backward_partial_dev(D[b0:b1], amax[b0:b1]))
                 for b0, b1 in zip(edges[:-1], edges[1:])]
        for b0, b1, P in parts:
            t.backward_finish_dev(P, amax[b0:b1], G[b0:b1])

    outs = []
    for chunks in (1, 4, 3):
        t = xb.AnalogTile(R, C, s, 21)
        t.set_stream(stream.cuda_stream)
        t.set_weights(W)
        g = torch.Generator(device="cuda").manual_seed(6)
        D = torch.rand(B, R, device="cuda", generator=g) * 2 - 1
        G1 = torch.empty(B, C, device="cuda")
        G2 = torch.empty(B, C, device="cuda")
        run(t, D, G1, chunks)
        run(t, D, G2, 1)
        torch.cuda.synchronize()
        outs.append((G1.cpu().numpy(), G2.cpu().numpy()))
    for G1, G2 in outs[1:]:
        np.testing.assert_array_equal(G1, outs[0][0])
        np.testing.assert_array_equal(G2, outs[0][1])
    assert not np.array_equal(outs[0][0], outs[0][1])  # fresh noise per call


def test_split_phase_backward_beyond_grid_y_limit():
    """More samples than a grid's y dimension holds (65535): the split-phase
    backward in one call equals the same entries in two chunks below the
    limit, bit for bit (the partial/finish kernels stride over samples)."""
    R, C, B = 24, 16, 70000
    bio = xb.default_io()
    s = xb.TileSettings(device=xb.device_preset("reram_sb"), backward_io=bio)
    W = np.random.default_rng(8).uniform(-0.3, 0.3, (R, C)).astype(np.float32)
    g = torch.Generator(device="cuda").manual_seed(6)
    D = torch.rand(B, R, device="cuda", generator=g) * 2 - 1
    out = []
    for edges in ((0, B), (0, 40000, B)):
        t = xb.AnalogTile(R, C, s, 21)
        t.set_stream(torch.cuda.current_stream().cuda_stream)
        t.set_weights(W)
        amax = t.rows_amax(D)
        G = torch.empty(B, C, device="cuda")
        for b0, b1 in zip(edges[:-1], edges[1:]):
            P = t.backward_partial_dev(D[b0:b1], amax[b0:b1])
            t.backward_finish_dev(P, amax[b0:b1], G[b0:b1])
        torch.cuda.synchronize()
        out.append(G.cpu().numpy())
    np.testing.assert_array_equal(out[0], out[1])
    assert np.abs(out[0]).max() > 0
