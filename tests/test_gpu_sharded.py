"""GPU check of the slice-sharded update (distributed.py) with two ranks
simulated in one process: each rank is a thread with its own StreamState,
dash context and CUDA stream on cuda:0; the all-reduce of the fresh F/G sums
is a host-side exchange summed in fixed rank order (what NCCL all-reduce
provides across GPUs).  This exercises the split entry points
dash_update_pass_begin / dash_update_pass_finish the multi-GPU bench uses.
Compared with one unsharded GPU state and with the CPU oracle."""
import threading

import numpy as np
import pytest
import torch

from golden_io import rel
from oracle import dash_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_18376_b200.build import build_library
    build_library()


class HostAllReduce:
    """Sum of both ranks' tensors, rank 0 + rank 1 (identical bytes on both)."""

    def __init__(self, world):
        self.world = world
        self.bar = threading.Barrier(world)
        self.buf = [None] * world

    def fn(self, rank):
        def allreduce(t):
            torch.cuda.current_stream().synchronize()
            self.buf[rank] = t.cpu()
            self.bar.wait()
            tot = self.buf[0].clone()
            for r in range(1, self.world):
                tot += self.buf[r]
            self.bar.wait()
            t.copy_(tot.to(t.device))
        return allreduce


def _rank_state(ps, owned, dtype):
    from paper_2305_18376_b200.stream import StreamState
    idx = {s: k for k, s in enumerate(ps["slice_ids"])}
    rows = np.array([idx[s] for s in owned], dtype=np.int64)
    arr = dict(ps, slice_ids=list(owned), W=ps["W"][rows], C=ps["C"][rows], D=ps["D"][rows])
    st = StreamState.from_arrays(arr, dtype=dtype)  # owns its context (workspace, plan), like a process
    return st


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_two_rank_sharded_gpu_update(dtype):
    from paper_2305_18376_b200 import workloads as wl
    from paper_2305_18376_b200.distributed import ShardedStream, owner_of_index
    from paper_2305_18376_b200.stream import StreamState
    world = 2
    cfg = wl.scaled(wl.CONFIGS["large"], K0=120, steps=3, new_slices=4)
    stream = wl.make_stream(cfg)
    ps = wl.planted_state(stream)
    batches = list(stream.batches())
    ids = ps["slice_ids"]
    ar = HostAllReduce(world)
    states, errs = {}, []

    def run(rank):
        try:
            owned = [s for k, s in enumerate(ids) if owner_of_index(k, world) == rank]
            st = _rank_state(ps, owned, dtype)
            eng = ShardedStream(st, rank, world, global_ids=ids, allreduce=ar.fn(rank))
            with torch.cuda.stream(torch.cuda.Stream()):
                for b in batches:
                    eng.update(b)
                torch.cuda.current_stream().synchronize()
            states[rank] = st
        except Exception as e:  # surfaced below
            errs.append(e)
            ar.bar.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    s0, s1 = states[0], states[1]
    for name in ("V", "F", "G"):  # replicated: bit-identical on both ranks
        assert np.array_equal(getattr(s0, name), getattr(s1, name)), name
    # against one unsharded GPU state and the CPU oracle
    one = StreamState.from_arrays(ps, dtype=dtype)
    R = cfg.R
    ref = orc.OracleStreamState(ps["slice_ids"], {s: [np.zeros((0, R))] for s in ps["slice_ids"]},
                                ps["W"], ps["V"], ps["C"], ps["D"], ps["F"], ps["G"], ps["forgetting"])
    for b in batches:
        one.update(b)
        ref.update(b)
    tol_one = 1e-12 if dtype == torch.float64 else 1e-6
    tol_ref = 1e-8 if dtype == torch.float64 else 1e-3
    for name in ("V", "F", "G"):
        assert rel(getattr(s0, name), getattr(one, name)) < tol_one, name
        assert rel(getattr(s0, name), getattr(ref, name)) < tol_ref, name
    for st in (s0, s1):
        for sid in st.slice_ids:
            k = ref.row_of(sid)
            for name in ("W", "C", "D"):
                a = getattr(st, name)[st.row_of(sid)]
                assert rel(a, getattr(ref, name)[k]) < tol_ref, (name, sid)
