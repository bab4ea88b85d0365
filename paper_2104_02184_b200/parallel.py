"""Row sharding of one logical analog tile over the ranks of a process group.

SURVEY.md §8e: rank r owns rows [r0, r1) of W and of every per-cell array.
Random draws are keyed on global indices, so P shards reproduce the
unsharded tile.  The only data-path collectives:

* update  : all-reduce(max) of the per-sample max|d| (translate needs the
            global value, proj/src/pulsed.cpp:34-51); x is replicated;
* backward: all-reduce(max) of max|d| before the DAC, then all-reduce(sum)
            of the per-shard column sums; output noise, ADC and alpha are
            applied after the reduction (proj/src/io.cpp:143-146);
* forward : none (outputs stay row-sharded).

The local compute object needs five methods (``forward_dev``,
``update_dev``, ``backward_partial_dev``, ``backward_finish_dev``,
``rows_amax``); on a B200 it is :class:`AnalogTile` built with ``shard=``.
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


class RowShardedTile:
    """One logical d_out x d_in tile, row-sharded over ``group``."""

    def __init__(self, local, d_out: int, d_in: int, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.rows = partition_rows(d_out, self.world, self.rank)
        self.local = local
        self.d_out, self.d_in = d_out, d_in

    @classmethod
    def create(cls, d_out: int, d_in: int, settings, seed: int, group=None):
        """Build the local B200 shard (``AnalogTile(shard=...)``) of this rank."""
        import torch.distributed as dist

        from .tile import AnalogTile
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        r0, r1 = partition_rows(d_out, world, rank)
        local = AnalogTile(d_out, d_in, settings, seed, shard=(r0, r1) if world > 1 else None)
        return cls(local, d_out, d_in, group)

    def _amax_global(self, D):
        amax = self.local.rows_amax(D)
        if self.world > 1:
            self.dist.all_reduce(amax, op=self.dist.ReduceOp.MAX, group=self.group)
        return amax

    def forward(self, X, Y, io=None):
        """Y[:, local rows] of the noisy forward; no collective."""
        self.local.forward_dev(X, Y, io)
        return Y

    def update(self, X, D_local, lr=None):
        """B sequential pulsed updates of the whole tile; D_local = this rank's rows of d."""
        self.local.update_dev(X, D_local, lr, amax_d=self._amax_global(D_local))

    def backward(self, D_local, G):
        """Full backward G[B][d_in] (replicated on every rank)."""
        amax = self._amax_global(D_local)
        P = self.local.backward_partial_dev(D_local, amax)
        if self.world > 1:
            self.dist.all_reduce(P, op=self.dist.ReduceOp.SUM, group=self.group)
        self.local.backward_finish_dev(P, amax, G)
        return G


__all__ = ["partition_rows", "RowShardedTile"]

