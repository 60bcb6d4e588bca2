"""Accumulated data on the GPU: the device X-history store
``DeviceTensor.apply_batch`` (tensor.py:228-244), the two-term accumulated
error ``global_error`` (evaluate.py:121-144) and the baseline refit
``parafac2_als(accumulated, tol=0.0)`` (evaluate.py:212-222), checked against
the host restatements / the oracle on the same seeded streams.
"""
import numpy as np
import pytest
import torch

from golden_io import rel
from oracle import dash_oracle as orc

pytestmark = pytest.mark.gpu

TOL = 1e-8


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _stream(K0=60, steps=4):
    from paper_2305_18376_b200 import workloads as wl
    cfg = wl.scaled(wl.CONFIGS["medium"], K0=K0, steps=steps)
    return wl.make_stream(cfg)


def test_device_apply_batch_matches_host_apply_batch():
    from paper_2305_18376_b200.history import DeviceTensor
    from paper_2305_18376_b200.tensor import DatasetError, NewSlice, UpdateBatch, apply_batch
    stream = _stream()
    host = stream.initial_tensor()
    dev = DeviceTensor.from_tensor(host, device="cuda")
    for batch in stream.batches():
        host = apply_batch(host, batch)
        dev = dev.apply_batch(batch)
        assert dev.slice_ids == host.slice_ids
        assert np.array_equal(np.diff(dev.row_ptr), [s.row_count for s in host.slices])
        assert np.array_equal(dev.X.cpu().numpy(), np.concatenate([s.rows for s in host.slices]))
    bad = UpdateBatch(99, {"nope": np.ones((1, dev.column_count))}, [NewSlice("fresh", np.ones((2, dev.column_count)), 99)],
                      (99, 99))
    with pytest.raises(DatasetError):
        dev.apply_batch(bad)


def test_baseline_refit_on_the_device_tensor_matches_host_and_oracle():
    from paper_2305_18376_b200.als import parafac2_als
    from paper_2305_18376_b200.history import DeviceTensor, refit_baseline
    from paper_2305_18376_b200.tensor import apply_batch
    stream = _stream(K0=40, steps=2)
    host = stream.initial_tensor()
    dev = DeviceTensor.from_tensor(host, device="cuda")
    for t, batch in enumerate(stream.batches()):
        host = apply_batch(host, batch)
        dev = dev.apply_batch(batch)
        seed = 7919 * (t + 1)
        fd = refit_baseline(dev, 10, iters=4, seed=seed)
        fh, ih = parafac2_als(host, 10, iters=4, seed=seed, tol=0.0, return_info=True)
        assert rel(fd.W, fh.W) < 1e-12 and rel(fd.V, fh.V) < 1e-12
        U, W, V, losses, _, _ = orc.parafac2_als([(s.slice_id, s.rows) for s in host.slices], 10, iters=4,
                                                 seed=seed, tol=0.0)
        assert len(ih.losses) == len(losses) == 4
        np.testing.assert_allclose(ih.losses, losses, rtol=TOL, atol=0)
        assert rel(fh.W, W) < TOL and rel(fh.V, V) < TOL


def test_global_error_matches_the_reference_formula():
    """run_experiment's track_global bookkeeping (evaluate.py:190-210): the
    retained rows of every pre-update slice with their pre-update row factors,
    plus the newest batch, under the post-update W and V."""
    from paper_2305_18376_b200 import workloads as wl
    from paper_2305_18376_b200.history import DeviceTensor, global_error, global_error_device
    from paper_2305_18376_b200.stream import initialize
    stream = _stream(K0=30, steps=3)
    init = stream.initial_tensor()
    state, _ = initialize(init, 10, iters=3, seed=0, forgetting=0.9)
    hist_host = {s.slice_id: s.rows for s in init.slices}
    hist_dev = DeviceTensor.from_tensor(init, device="cuda")
    for batch in stream.batches():
        old_factors = {sid: state.u_matrix(sid) for sid in state.slice_ids}
        U_hist = state.u_history_device(hist_dev.slice_ids)
        res = state.update(batch)
        items = [(sid, rows) for sid, rows, _ in batch.items()]
        w_rows = {sid: state.W[state.row_of(sid)] for sid in state.slice_ids}
        want = orc.global_error(hist_host, old_factors, dict(items), {s: res.u_new[s] for s, _ in items},
                                w_rows, state.V)
        got_dict = global_error(hist_host, old_factors, dict(items), dict(res.u_new), w_rows, state.V)
        got_dev = global_error_device(hist_dev, U_hist, state, items, res.u_new)
        assert abs(got_dict - want) <= 1e-12 * abs(want)
        assert abs(got_dev - want) <= 1e-12 * abs(want)
        for sid, rows in items:  # history after the update (evaluate.py:224-227)
            prev = hist_host.get(sid)
            hist_host[sid] = rows if prev is None else np.vstack([prev, rows])
        hist_dev = hist_dev.apply_batch(batch)
    del wl
