"""Row sharding of one logical analog tile over the ranks of a process group.

SURVEY.md §8e: rank r owns rows [r0, r1) of W and of every per-cell array.
Random draws are keyed on global indices, so P shards reproduce the
unsharded tile.  The only data-path collectives:

* update  : all-reduce(max) of the per-sample max|d| (translate needs the
            global value, proj/src/pulsed.cpp:34-51); x is replicated;
* backward: all-reduce(max) of max|d| before the DAC, then all-reduce(sum)
            of the per-shard column sums, in sample chunks whose reductions
            overlap the next chunk's contraction; output noise, ADC and alpha
            are applied after the reduction (proj/src/io.cpp:143-146);
* forward : none (outputs stay row-sharded).

The local compute object needs five methods (``forward_dev``,
``update_dev``, ``backward_partial_dev``, ``backward_finish_dev``,
``rows_amax``); on a B200 it is :class:`AnalogTile` built with ``shard=``,
running on the torch stream current at the calls
(``local.set_stream(torch.cuda.current_stream().cuda_stream)``): the NCCL
collectives are ordered after the tile's kernels through that stream.
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
        # the NCCL collectives are issued on torch's current stream: the tile
        # must run on that same stream, or a reduction could read a buffer
        # before the tile's kernel has written it (and vice versa)
        bind = getattr(local, "set_stream", None)
        if bind is not None:
            import torch
            if torch.cuda.is_available():
                bind(torch.cuda.current_stream().cuda_stream)

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

    def backward(self, D_local, G, chunks: int | None = None):
        """Full backward G[B][d_in] (replicated on every rank).

        The batch is cut into ``chunks`` sample ranges (default: 4 when every
        range keeps >= 64 samples, else 1): all chunk contractions are issued
        back to back, each followed by its asynchronous all-reduce(sum), so
        the reduction of chunk c overlaps the contraction of chunk c + 1;
        the finishes (noise, ADC, alpha) then run in chunk order.  The noise
        draws are addressed by sample, so every chunking gives the same G."""
        amax = self._amax_global(D_local)
        B = int(D_local.shape[0])
        n = chunks if chunks is not None else (4 if B >= 256 else 1)
        n = max(1, min(n, B))
        edges = [B * k // n for k in range(n + 1)]
        inflight = []
        for b0, b1 in zip(edges[:-1], edges[1:]):
            if b1 == b0:
                continue
            P = self.local.backward_partial_dev(D_local[b0:b1], amax[b0:b1])
            work = None
            if self.world > 1:
                work = self.dist.all_reduce(P, op=self.dist.ReduceOp.SUM, group=self.group,
                                            async_op=True)
            inflight.append((b0, b1, P, work))
        for b0, b1, P, work in inflight:
            if work is not None:
                work.wait()
            self.local.backward_finish_dev(P, amax[b0:b1], G[b0:b1])
        return G


__all__ = ["partition_rows", "RowShardedTile"]

