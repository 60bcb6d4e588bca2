"""World-size-2 gloo test of the slice-sharded update protocol
(paper_2305_18376_b200/distributed.py) on CPU.

Each rank owns a subset of slices; per pass it computes the fresh F/G sums of
its own slices, the sums are all-reduced, and every rank forms F, G and solves
V.  The per-shard math here is the CPU oracle (test infrastructure) standing in
for the device kernel; what is under test is the host protocol -- ownership,
registration order, the all-reduce placement and decay -- which must reproduce
the single-process reference update exactly (up to reduction order).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import dash_oracle as orc


class OracleShard:
    """CPU stand-in for a rank's StreamState: same _update_items contract."""

    def __init__(self, ps, owned_ids):
        self.R = ps["V"].shape[1]
        self.lam = ps["forgetting"]
        self.V, self.F, self.G = ps["V"].copy(), ps["F"].copy(), ps["G"].copy()
        idx = {s: k for k, s in enumerate(ps["slice_ids"])}
        self.W = {s: ps["W"][idx[s]].copy() for s in owned_ids}
        self.C = {s: ps["C"][idx[s]].copy() for s in owned_ids}
        self.D = {s: ps["D"][idx[s]].copy() for s in owned_ids}
        self.passes = 1

    def _update_items(self, entries, allreduce):
        R, lam = self.R, self.lam
        F0, G0 = self.F.copy(), self.G.copy()
        snap = {}
        for sid, rows, is_new in entries:
            if is_new:
                self.W[sid] = np.ones(R)
                self.C[sid] = np.zeros(R)
                self.D[sid] = np.zeros((R, R))
            snap[sid] = (self.C[sid].copy(), self.D[sid].copy())
        for _ in range(self.passes):
            vtv = self.V.T @ self.V
            f = np.zeros_like(F0)
            g = np.zeros_like(G0)
            res = {}
            for sid, rows, _ in entries:
                xv = (rows @ self.V)[None]
                u, us, c_new, d_new, w, gf, ok = orc.group_update(
                    xv, vtv, self.W[sid][None], snap[sid][0][None], snap[sid][1][None], lam, orc.RIDGE_EPS)
                f += rows.T @ us[0]
                g += gf
                self.W[sid] = w[0]
                res[sid] = (c_new[0], d_new[0])
            fg = torch.from_numpy(np.concatenate([f.ravel(), g.ravel()]))
            allreduce(fg)
            fg = fg.numpy()
            J = F0.shape[0]
            self.F = lam * F0 + fg[:J * R].reshape(J, R)
            self.G = orc.symmetrize(lam * G0 + fg[J * R:].reshape(R, R))
            self.V = orc.ridge_solve(self.G, self.F.T).T
        for sid, (c, d) in res.items():
            self.C[sid], self.D[sid] = c, d


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2305_18376_b200 import workloads as wl
    from paper_2305_18376_b200.distributed import ShardedStream, owner_of_index
    orc.build_c()
    cfg = wl.scaled(wl.CONFIGS["medium"], K0=30, steps=3, new_slices=3)
    stream = wl.make_stream(cfg)
    ps = wl.planted_state(stream)
    ids = ps["slice_ids"]
    owned = [s for k, s in enumerate(ids) if owner_of_index(k, world) == rank]
    shard = OracleShard(ps, owned)
    eng = ShardedStream(shard, rank, world, global_ids=ids,
                        allreduce=lambda t: dist.all_reduce(t))
    for b in stream.batches():
        eng.update(b)
    out[rank] = {"V": shard.V, "F": shard.F, "G": shard.G, "W": dict(shard.W)}
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_sharded_update_equals_single_process():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    from paper_2305_18376_b200 import workloads as wl
    cfg = wl.scaled(wl.CONFIGS["medium"], K0=30, steps=3, new_slices=3)
    stream = wl.make_stream(cfg)
    ps = wl.planted_state(stream)
    R = cfg.R
    ref = orc.OracleStreamState(ps["slice_ids"], {s: [np.zeros((0, R))] for s in ps["slice_ids"]},
                                ps["W"], ps["V"], ps["C"], ps["D"], ps["F"], ps["G"], ps["forgetting"])
    for b in stream.batches():
        ref.update(b)
    r0, r1 = out[0], out[1]
    # replicated factors identical on both ranks, and equal to the single-process run
    assert np.array_equal(r0["V"], r1["V"])
    for name in ("V", "F", "G"):
        a, b = r0[name], getattr(ref, name)
        assert np.abs(a - b).max() / np.abs(b).max() < 1e-12, name
    # every slice owned by exactly one rank, with the reference's W row
    allw = dict(r0["W"])
    assert not set(allw) & set(r1["W"])
    allw.update(r1["W"])
    assert set(allw) == set(ref.slice_ids)
    for sid, w in allw.items():
        want = ref.W[ref.row_of(sid)]
        assert np.abs(w - want).max() <= 1e-12 * max(1.0, np.abs(want).max())


def test_new_slices_go_to_the_least_loaded_rank_deterministically():
    """a new slice lands on the rank with the fewest rows in the update that brings it
    (ties: fewer owned slices, then the lowest rank); every rank computes the same map."""
    from paper_2305_18376_b200.distributed import Placement, place_counts
    world = 4
    ids = [f"s{k}" for k in range(10)]
    rng = np.random.default_rng(0)
    maps = []
    for _ in range(2):  # two "ranks" replaying the same batches
        pl = Placement(world, ids)
        assert [pl.owner[s] for s in ids] == [k % world for k in range(10)]
        r2 = np.random.default_rng(1)
        known = list(ids)
        for t in range(5):
            ex = [(s, int(r2.integers(1, 9))) for s in known]
            new = [(f"n{t}_{i}", int(r2.integers(200, 2001))) for i in range(6)]
            owners = pl.place(ex, new)
            # replay the rule by hand
            load = [0] * world
            for s, n in ex:
                load[pl.owner[s]] += n
            # (owners were appended in order; check each choice was a minimum at its time)
            own_cnt = [sum(1 for s in known if pl.owner[s] == q) for q in range(world)]
            for (s, n), r in zip(new, owners):
                assert (load[r], own_cnt[r], r) == min((load[q], own_cnt[q], q) for q in range(world))
                load[r] += n
                own_cnt[r] += 1
            known += [s for s, _ in new]
            # per-update rows end up balanced to within one new slice
            assert max(load) - min(load) <= 2000
        maps.append(dict(pl.owner))
    assert maps[0] == maps[1]
    # index form used by bench.py agrees with the id form
    pl = Placement(2, ["a", "b", "c"])
    got = place_counts(2, list(pl.n_owned), [5, 1], [10, 3, 3])
    assert list(got) == pl.place([("a", 3), ("b", 1), ("c", 2)], [("x", 10), ("y", 3), ("z", 3)])
