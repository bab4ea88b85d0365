"""Row-sharded tiles through the library's communicators (include/xbtile.h,
xb_comm_*): P shard handles of one logical tile, each driven by its own host
thread (as one process per GPU would), joined by an in-process loopback
group on the one GPU of the test box; and the NCCL communicator itself
(dlopen'd libnccl) on a one-rank group.  Invariants:
update and forward (bound management on, saturation flags all-reduced) are
bit-identical to the unsharded tile; the backward differs only by the fp32
order of the cross-rank sum (<= 1 ADC LSB)."""
import threading

import numpy as np
import pytest
import torch

import paper_2104_02184_b200 as xb
from paper_2104_02184_b200.parallel import RowShardedTile, partition_rows

pytestmark = pytest.mark.gpu


def run_ranks(P, fn):
    """fn(rank) on P host threads; re-raises the first failure."""
    errs = [None] * P

    def body(r):
        try:
            fn(r)
        except BaseException as e:  # noqa: BLE001
            errs[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in errs:
        if e is not None:
            raise e


def settings(prec, bm):
    io = xb.default_io()
    io.sigma_w = 0.01
    io.bound_management = xb.BM_ITERATIVE if bm else xb.BM_NONE
    bio = xb.default_io()
    return xb.TileSettings(device=xb.device_preset("reram_sb"), forward_io=io, backward_io=bio,
                           mvm_precision=prec)


@pytest.mark.parametrize("P,R,C,B,prec", [(2, 1024, 512, 256, xb.MVM_TF32),
                                          (3, 520, 300, 40, xb.MVM_TF32X3),
                                          (2, 200, 96, 33, xb.MVM_FP32)])
def test_loopback_group_reproduces_unsharded_tile(P, R, C, B, prec):
    cfg = settings(prec, bm=True)
    r = np.random.default_rng(11)
    # weights large enough that bound management re-issues samples
    W = r.uniform(-0.5, 0.5, (R, C)).astype(np.float32)
    X = r.uniform(-1, 1, (B, C)).astype(np.float32)
    D = r.uniform(-1, 1, (B, R)).astype(np.float32)
    X2 = r.uniform(-1, 1, (B, C)).astype(np.float32)

    full = xb.AnalogTile(R, C, cfg, 99)
    full.set_weights(W)
    Yf = full.forward(X)
    Gf = full.backward(D)
    full.update(X, D, 0.01)
    Yf2 = full.forward(X2)
    Wf = full.get_weights()

    comms = xb.Comm.local(P)
    out = [None] * P

    def rank(q):
        r0, r1 = partition_rows(R, P, q)
        t = xb.AnalogTile(R, C, cfg, 99, shard=(r0, r1))
        t.attach_comm(comms[q])
        t.set_weights(W[r0:r1])
        y = t.forward(X)            # bound management: flags all-reduced per pass
        g = t.backward(D[:, r0:r1])  # max|d| and column sums all-reduced
        t.update(X, D[:, r0:r1], 0.01)  # global max|d| for translate
        y2 = t.forward(X2)
        out[q] = (y, g, t.get_weights(), y2)

    run_ranks(P, rank)
    Ys = np.hstack([o[0] for o in out])
    np.testing.assert_array_equal(Ys, Yf)
    np.testing.assert_array_equal(np.vstack([o[2] for o in out]), Wf)
    np.testing.assert_array_equal(np.hstack([o[3] for o in out]), Yf2)
    lsb = (2 * 12.0 / 512) * np.abs(D).max(axis=1)[:, None]
    for o in out:  # every rank holds the full G
        np.testing.assert_array_equal(o[1], out[0][1])
        diff = np.abs(o[1] - Gf)
        assert np.all(diff <= lsb * 1.001 + 1e-6)
        assert np.mean(diff > 1e-6) < 0.02


def test_row_sharded_tile_api_loopback():
    """parallel.RowShardedTile over a loopback group, device-pointer calls on
    each shard's stream (the path bench.py --gpus N takes with NCCL)."""
    P, R, C, B = 2, 512, 256, 64
    cfg = settings(xb.MVM_TF32, bm=False)
    W = np.random.default_rng(3).uniform(-0.2, 0.2, (R, C)).astype(np.float32)
    g = torch.Generator(device="cuda").manual_seed(4)
    X = torch.rand(B, C, device="cuda", generator=g) * 2 - 1
    D = torch.rand(B, R, device="cuda", generator=g) * 2 - 1
    full = xb.AnalogTile(R, C, cfg, 5)
    full.set_weights(W)
    full.update_dev(X, D, 0.01)
    full.synchronize()
    comms = xb.Comm.local(P)
    res = [None] * P

    def rank(q):
        sh = RowShardedTile.create(R, C, cfg, 5, comms[q])
        r0, r1 = sh.rows
        sh.local.set_weights(W[r0:r1])
        sh.update(X, D[:, r0:r1].contiguous(), 0.01)
        sh.local.synchronize()
        res[q] = sh.local.get_weights()

    run_ranks(P, rank)
    np.testing.assert_array_equal(np.vstack(res), full.get_weights())


def test_nccl_communicator_single_rank():
    """The NCCL path itself (dlopen, ncclGetUniqueId, ncclCommInitRank,
    ncclAllReduce) on a one-rank group: a 1-shard tile with the NCCL comm
    attached equals the plain tile."""
    R, C, B = 256, 128, 32
    cfg = settings(xb.MVM_TF32, bm=True)
    uid = xb.Comm.unique_id()
    assert len(uid) == 128
    comm = xb.Comm(uid, 1, 0)
    assert (comm.size, comm.rank) == (1, 0)
    a = xb.AnalogTile(R, C, cfg, 8, shard=(0, R))
    a.attach_comm(comm)
    b = xb.AnalogTile(R, C, cfg, 8)
    W = np.random.default_rng(1).uniform(-0.4, 0.4, (R, C)).astype(np.float32)
    for t in (a, b):
        t.set_weights(W)
    X = np.random.default_rng(2).uniform(-1, 1, (B, C)).astype(np.float32)
    D = np.random.default_rng(3).uniform(-1, 1, (B, R)).astype(np.float32)
    for t in (a, b):
        t.update(X, D, 0.02)
    np.testing.assert_array_equal(a.forward(X), b.forward(X))
    np.testing.assert_array_equal(a.get_weights(), b.get_weights())


def test_attach_requires_a_shard():
    comms = xb.Comm.local(2)
    t = xb.AnalogTile(64, 32, settings(xb.MVM_FP32, False), 1)
    with pytest.raises(xb.Error, match="not row-sharded"):
        t.attach_comm(comms[0])
