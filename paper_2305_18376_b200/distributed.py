"""Slice-sharded DASH updates over torch.distributed (one process per GPU).

Partitioning: every slice has one owner rank; its per-slice
state (W/C/D rows, U history) lives only there.  V, F, G are replicated.  Per
pass each rank runs the per-slice phase on its own slices and produces the
fresh sums [f (J x R) | g (R x R)]; one all-reduce (NCCL over NVLink, the
only data-path collective) combines them, and every rank then forms F, G and
solves V redundantly -- the all-reduce returns identical bytes on every rank,
so V stays bit-identical across ranks.

Ownership is deterministic and computed identically on every
rank from the batches alone:
  * initial slices: by position (k % world) -- their appends are identically
    distributed, so balancing by count balances expected rows;
  * new slices: each goes to the rank with the least rows in the update that
    brings it (existing slices' rows first, then the new slices in batch
    order -- a new slice is 100-2,000 rows against 1-8 for an existing one, so
    this is what decides the per-update imbalance); ties go to the rank that
    owns fewer slices, then to the lowest rank.
"""
from __future__ import annotations

import numpy as np


def owner_of_index(k: int, world: int) -> int:
    """Owner of the k-th INITIAL slice."""
    return k % world


class Placement:
    """Slice -> owner map shared by every rank (same inputs, same answers)."""

    def __init__(self, world: int, initial_ids=()):
        self.world = world
        self.owner: dict = {}
        self.n_owned = [0] * world
        for k, sid in enumerate(initial_ids):
            r = owner_of_index(k, world)
            self.owner[sid] = r
            self.n_owned[r] += 1

    def place(self, existing, new):
        """``existing``: (sid, rows) of the batch's existing slices, ``new``:
        (sid, rows) of its new slices in batch order.  Registers the new
        slices and returns their owners."""
        load = [0] * self.world
        for sid, n in existing:
            load[self.owner[sid]] += int(n)
        out = []
        for sid, n in new:
            r = min(range(self.world), key=lambda q: (load[q], self.n_owned[q], q))
            self.owner[sid] = r
            self.n_owned[r] += 1
            load[r] += int(n)
            out.append(r)
        return out


def place_counts(world: int, n_owned, existing_load, new_counts):
    """Index form of Placement.place for packed batches (bench): per-rank
    existing-row loads and owned-slice counts in, owners of the new slices
    out; ``n_owned`` is updated in place."""
    load = [int(v) for v in existing_load]
    out = np.empty(len(new_counts), dtype=np.int64)
    for i, n in enumerate(new_counts):
        r = min(range(world), key=lambda q: (load[q], n_owned[q], q))
        n_owned[r] += 1
        load[r] += int(n)
        out[i] = r
    return out


class ShardedStream:
    """Wraps this rank's ``StreamState`` (holding only owned slices)."""

    def __init__(self, state, rank: int, world: int, group=None, global_ids=None,
                 allreduce=None):
        self.state = state
        self.rank = rank
        self.world = world
        self.group = group
        # slice -> owner, built identically on every rank (initial slices by position)
        self.placement = Placement(world, global_ids or [])
        self._allreduce = allreduce or self._nccl_allreduce

    @property
    def dtype(self):
        """Streamed-data dtype of the wrapped state (FP64, or FP32 data mode)."""
        return self.state.dtype

    def _nccl_allreduce(self, t):
        import torch.distributed as dist
        dist.all_reduce(t, group=self.group)

    def owns(self, sid) -> bool:
        return self.placement.owner[sid] == self.rank

    def split(self, batch):
        """This rank's entries of a global UpdateBatch, in batch order."""
        owner = self.placement.owner
        items = list(batch.items())
        for sid, _, is_new in items:
            if is_new and sid in owner:
                raise ValueError(f"batch declares known slice {sid!r} as new")
            if not is_new and sid not in owner:
                raise ValueError(f"batch references unknown existing slice {sid!r}")
        self.placement.place([(sid, rows.shape[0]) for sid, rows, new in items if not new],
                             [(sid, rows.shape[0]) for sid, rows, new in items if new])
        return [(sid, rows, is_new) for sid, rows, is_new in items if owner[sid] == self.rank]

    def update(self, batch):
        """Global batch in, this rank's UpdateResult out (u_new holds only the
        owned slices; V/F/G identical on every rank)."""
        return self.state._update_items(self.split(batch), allreduce=self._allreduce)

    def update_packed(self, X, counts, existing_rows, new_ids, check=False):
        """Local shard already packed on this GPU (bench path)."""
        return self.state.update_packed(X, counts, np.asarray(existing_rows, dtype=np.int32),
                                        new_ids, check=check, allreduce=self._allreduce)
