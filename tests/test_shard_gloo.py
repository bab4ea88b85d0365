"""World-size-2 gloo tests of the row-sharding orchestration (CPU).

* the NCCL bootstrap (parallel.share_unique_id): rank 0's 128-byte unique id
  reaches every rank over a torch.distributed group;
* the sharding algebra the C library implements (include/xbtile.h, "row
  sharding"; csrc/xb_comm.cu): all-reduce(max) of max|d| before translate,
  all-reduce(sum) of the per-shard column sums (in in-flight sample chunks,
  finished in order), row-local forward.  The collectives run over gloo
  between two processes; the per-shard compute is a test double restating
  the deterministic, noise-free tile in numpy (ConstantStep,
  deterministic_implicit pulses, perfect IO) -- test infrastructure, not a
  product fallback -- and the sharded result must equal the unsharded oracle
  tile.  The same orchestration on the device is tests/test_gpu_comm.py."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2104_02184_b200.parallel import partition_rows, share_unique_id

R, C, B, LR, DW = 13, 9, 6, 0.05, 0.01


class NumpyShard:
    """Deterministic-mode restatement of one shard (proj/src/pulsed.cpp:25-66,128-144)."""

    def __init__(self, W, r0, r1):
        self.W = W[r0:r1].copy()

    def rows_amax(self, D):
        return torch.from_numpy(np.abs(D.numpy()).max(axis=1).astype(np.float64))

    def forward_dev(self, X, Y, io=None):
        Y[:] = torch.from_numpy(X.numpy() @ self.W.T)

    def update_dev(self, X, D, lr, amax_d):
        for b in range(X.shape[0]):
            x, d, dm = X[b].numpy(), D[b].numpy(), float(amax_d[b])
            xm = np.abs(x).max()
            if lr == 0 or xm == 0 or dm == 0:
                continue
            bl = 31
            amp = np.sqrt(lr / (DW * bl))
            xs = np.sqrt(dm / xm)
            px = np.minimum(1.0, amp * np.abs(x) * xs)
            pd = np.minimum(1.0, amp * np.abs(d) * (1.0 / xs))
            cnt = np.floor(bl * pd[:, None] * px[None, :] + 0.5)  # lround, non-negative
            self.W += DW * cnt * np.sign(d)[:, None] * np.sign(x)[None, :]

    def backward_partial_dev(self, D, amax_d):
        return torch.from_numpy(D.numpy() @ self.W)

    def backward_finish_dev(self, P, amax_d, G):
        G[:] = P


class ShardedOrchestration:
    """The C library's sharded-tile control flow (csrc/xb_abi.cu:
    update_device / backward_sharded; csrc/xb_mvm.cu: row-local forward),
    restated over torch.distributed for this CPU test."""

    def __init__(self, local):
        self.local = local

    def _amax(self, D):
        a = self.local.rows_amax(D)
        dist.all_reduce(a, op=dist.ReduceOp.MAX)
        return a

    def update(self, X, D_local, lr):
        self.local.update_dev(X, D_local, lr, amax_d=self._amax(D_local))

    def backward(self, D_local, G, chunks=1):
        amax = self._amax(D_local)
        B_ = D_local.shape[0]
        edges = [B_ * k // chunks for k in range(chunks + 1)]
        inflight = []
        for b0, b1 in zip(edges[:-1], edges[1:]):
            P = self.local.backward_partial_dev(D_local[b0:b1], amax[b0:b1])
            inflight.append((b0, b1, P, dist.all_reduce(P, async_op=True)))
        for b0, b1, P, work in inflight:
            work.wait()
            self.local.backward_finish_dev(P, amax[b0:b1], G[b0:b1])

    def forward(self, X, Y):
        self.local.forward_dev(X, Y)


def _worker(rank, world, port, W, X, D, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    uid = share_unique_id(lambda: bytes(range(128)))
    assert uid == bytes(range(128))
    r0, r1 = partition_rows(R, world, rank)
    t = ShardedOrchestration(NumpyShard(W, r0, r1))
    Dl = torch.from_numpy(D[:, r0:r1].copy())
    Xt = torch.from_numpy(X)
    t.update(Xt, Dl, LR)
    G = torch.zeros(B, C, dtype=torch.float64)
    t.backward(Dl, G)
    G3 = torch.zeros(B, C, dtype=torch.float64)
    t.backward(Dl, G3, chunks=3)  # three in-flight async all-reduces, finished in order
    Y = torch.zeros(B, r1 - r0, dtype=torch.float64)
    t.forward(Xt, Y)
    out[rank] = (t.local.W.copy(), G.numpy().copy(), Y.numpy().copy(), G3.numpy().copy())
    dist.destroy_process_group()


def test_partition_rows():
    assert [partition_rows(10, 3, r) for r in range(3)] == [(0, 4), (4, 7), (7, 10)]
    assert partition_rows(4096 * 8, 8, 7) == (7 * 4096, 8 * 4096)
    with pytest.raises(ValueError):
        partition_rows(2, 3, 0)


def test_two_rank_gloo_matches_unsharded_oracle():
    rng = np.random.default_rng(0)
    W = rng.uniform(-0.1, 0.1, (R, C))
    X = rng.uniform(-1, 1, (B, C))
    D = rng.uniform(-1, 1, (B, R))
    D[:, 7:] *= 3.0  # the global max|d| lives on rank 1: translate must see it on rank 0 too
    mgr = mp.Manager()
    out = mgr.dict()
    port = 29500 + os.getpid() % 1000
    mp.spawn(_worker, args=(2, port, W, X, D, out), nprocs=2, join=True)
    Wsh = np.vstack([out[0][0], out[1][0]])

    O = oracle.load("restatement")
    s = O.default("tile")
    s.device.dw_min, s.device.w_max, s.device.w_min = DW, 10.0, -10.0
    s.update.pulse_type = oracle.PULSE_DETERMINISTIC
    s.forward_io = O.default("perfect_io")
    s.backward_io = O.default("perfect_io")
    o = O.tile(R, C, s, 1)
    o.set_weights(W)
    for b in range(B):
        o.update(X[b], D[b], LR)
    np.testing.assert_allclose(Wsh, o.get_weights(), rtol=0, atol=1e-12)
    Wo = o.get_weights()
    np.testing.assert_allclose(out[0][1], D @ Wo, atol=1e-12)  # replicated backward
    np.testing.assert_allclose(out[1][1], D @ Wo, atol=1e-12)
    np.testing.assert_array_equal(out[0][3], out[0][1])  # chunked = one-shot backward
    np.testing.assert_array_equal(out[1][3], out[1][1])
    np.testing.assert_allclose(np.hstack([out[0][2], out[1][2]]), X @ Wo.T, atol=1e-12)
