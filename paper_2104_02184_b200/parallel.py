"""Row sharding of one logical analog tile over several GPUs.

Rank r owns rows [r0, r1) of W and of every per-cell array
(:func:`partition_rows`).  The compute AND the collectives live in the C
library: each rank's :class:`~paper_2104_02184_b200.AnalogTile` is created
with ``shard=(r0, r1)`` and an attached :class:`~paper_2104_02184_b200.Comm`
(NCCL over NVLink/NVSwitch, ``xb_comm_create``), and then runs the whole-tile
semantics on its rows with every cross-rank reduction enqueued on its own
stream (include/xbtile.h, "row sharding"):

* update  : all-reduce(max) of the per-sample max|d| (translate needs the
            global value, proj/src/pulsed.cpp:34-51); x is replicated;
* forward : all-reduce(max) of the bound-management saturation flags before
            every re-issue; outputs stay row-sharded;
* backward: all-reduce(max) of max|d|, all-reduce(sum) of the column sums in
            sample chunks overlapping the next chunk's contraction; output
            noise, ADC and alpha after the sum (proj/src/io.cpp:143-146).

Random draws are keyed on global rows, so P shards reproduce the unsharded
tile (update and forward bit for bit).  Python only bootstraps: the NCCL
unique id travels from rank 0 to the others over an existing
``torch.distributed`` group (any backend, CPU objects), after which no
PyTorch collective is involved.
"""
from __future__ import annotations


def partition_rows(d_out: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced row ranges; the first d_out % world ranks get one more."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("partition_rows: need 0 <= rank < world")
    if d_out < world:
        raise ValueError(f"partition_rows: {d_out} rows cannot be split over {world} ranks")
    base, extra = divmod(d_out, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def share_unique_id(make_id, group=None) -> bytes:
    """Rank 0 calls ``make_id()`` (``Comm.unique_id``); every rank returns it.
    Bootstrap only: one 128-byte object over the torch.distributed group."""
    import torch.distributed as dist
    obj = [make_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def nccl_comm(group=None):
    """The NCCL communicator of this rank over ``group`` (current CUDA device)."""
    import torch.distributed as dist

    from .tile import Comm
    uid = share_unique_id(Comm.unique_id, group)
    return Comm(uid, dist.get_world_size(group), dist.get_rank(group))


class RowShardedTile:
    """One logical d_out x d_in tile, row-sharded over the ranks of ``comm``.

    ``local`` is this rank's shard handle (``AnalogTile(..., shard=rows)``);
    the communicator is attached to it here.  All calls take CUDA tensors
    (device pointers) and are asynchronous on the shard's stream."""

    def __init__(self, local, d_out: int, d_in: int, comm):
        self.local = local
        self.comm = comm
        self.world, self.rank = comm.size, comm.rank
        self.rows = partition_rows(d_out, self.world, self.rank)
        self.d_out, self.d_in = d_out, d_in
        if self.world > 1:
            local.attach_comm(comm)

    @classmethod
    def create(cls, d_out: int, d_in: int, settings, seed: int, comm):
        from .tile import AnalogTile
        r0, r1 = partition_rows(d_out, comm.size, comm.rank)
        shard = (r0, r1) if comm.size > 1 else None
        return cls(AnalogTile(d_out, d_in, settings, seed, shard=shard), d_out, d_in, comm)

    def forward(self, X, Y, io=None):
        """Y[:, local rows] of the noisy forward (x replicated on every rank)."""
        self.local.forward_dev(X, Y, io)
        return Y

    def update(self, X, D_local, lr=None):
        """B sequential pulsed updates of the whole tile; D_local = this rank's rows of d."""
        self.local.update_dev(X, D_local, lr)

    def backward(self, D_local, G):
        """Full backward G[B][d_in] (the same on every rank) from this rank's rows of d."""
        self.local.backward_dev(D_local, G)
        return G


__all__ = ["partition_rows", "share_unique_id", "nccl_comm", "RowShardedTile"]
