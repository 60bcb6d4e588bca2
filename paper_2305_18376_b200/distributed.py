"""Slice-sharded DASH updates over torch.distributed (one process per GPU).

Partitioning: every slice has one owner rank; its per-slice
state (W/C/D rows, U history) lives only there.  V, F, G are replicated.  Per
pass each rank runs the per-slice phase on its own slices and produces the
fresh sums [f (J x R) | g (R x R)]; one all-reduce (NCCL over NVLink, the
only data-path collective) combines them, and every rank then forms F, G and
solves V redundantly -- the all-reduce returns identical bytes on every rank,
so V stays bit-identical across ranks.

Ownership is deterministic and computed identically on every rank from the
batch alone: initial slices by position (k % world), new slices by their
global registration index.
"""
from __future__ import annotations

import numpy as np


def owner_of_index(k: int, world: int) -> int:
    return k % world


class ShardedStream:
    """Wraps this rank's ``StreamState`` (holding only owned slices)."""

    def __init__(self, state, rank: int, world: int, group=None, global_ids=None,
                 allreduce=None):
        self.state = state
        self.rank = rank
        self.world = world
        self.group = group
        # global registration order (needed to place new slices)
        self._global = {sid: i for i, sid in enumerate(global_ids or [])}
        self._allreduce = allreduce or self._nccl_allreduce

    @property
    def dtype(self):
        """Streamed-data dtype of the wrapped state (FP64, or FP32 data mode)."""
        return self.state.dtype

    def _nccl_allreduce(self, t):
        import torch.distributed as dist
        dist.all_reduce(t, group=self.group)

    def owns(self, sid) -> bool:
        return owner_of_index(self._global[sid], self.world) == self.rank

    def split(self, batch):
        """This rank's entries of a global UpdateBatch, in batch order."""
        local = []
        for sid, rows, is_new in batch.items():
            if is_new:
                if sid in self._global:
                    raise ValueError(f"batch declares known slice {sid!r} as new")
                self._global[sid] = len(self._global)
            elif sid not in self._global:
                raise ValueError(f"batch references unknown existing slice {sid!r}")
            if self.owns(sid):
                local.append((sid, rows, is_new))
        return local

    def update(self, batch):
        """Global batch in, this rank's UpdateResult out (u_new holds only the
        owned slices; V/F/G identical on every rank)."""
        return self.state._update_items(self.split(batch), allreduce=self._allreduce)

    def update_packed(self, X, counts, existing_rows, new_ids, check=False):
        """Local shard already packed on this GPU (bench path)."""
        return self.state.update_packed(X, counts, np.asarray(existing_rows, dtype=np.int32),
                                        new_ids, check=check, allreduce=self._allreduce)
