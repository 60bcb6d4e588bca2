"""GPU parity of the FP32 data mode (north_star's optional FP32 mode, reported
separately): X in and U_new out in FP32, state and arithmetic FP64
(``dash_update_f32``).

Two bars, both normwise (max|a-b| / max|b|) against the CPU oracle:
  * TOL_F32 = 1e-3 against the FP64 oracle on the original FP64 data (the
    north_star FP32 tolerance);
  * TOL_ROUNDED = 1e-5 against the FP64 oracle fed the FP32-rounded data: the
    kernels add no FP32 arithmetic error of their own beyond rounding U_new.
"""
import numpy as np
import pytest
import torch

from golden_io import rel
from oracle import dash_oracle as orc

pytestmark = pytest.mark.gpu

TOL_F32 = 1e-3
TOL_ROUNDED = 1e-5


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_18376_b200.build import build_library
    build_library()


def _round_batch(batch):
    from paper_2305_18376_b200.tensor import NewSlice, UpdateBatch
    f = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)  # noqa: E731
    return UpdateBatch(batch.update_index, {k: f(v) for k, v in batch.existing_rows.items()},
                       [NewSlice(ns.slice_id, f(ns.rows), ns.first_time_step) for ns in batch.new_slices],
                       batch.cycle_span)


def _oracle(ps, passes):
    R = ps["V"].shape[1]
    return orc.OracleStreamState(ps["slice_ids"], {s: [np.zeros((0, R))] for s in ps["slice_ids"]},
                                 ps["W"], ps["V"], ps["C"], ps["D"], ps["F"], ps["G"],
                                 ps["forgetting"], passes=passes)


@pytest.mark.parametrize("name,kw", [
    ("large", dict(K0=120, steps=3, new_slices=3)),   # R=16, J=128: float tensor-map GEMMs
    ("medium", dict(K0=150, steps=3)),                # R=10, J=88: tensor-map path, 3 float strips
    ("daily", dict(K0=300, steps=4)),                 # short new slices (n_k < R)
    ("wide32", dict(K0=40, steps=2, new_slices=2)),   # R=32: generic FP32-input GEMMs
    ("wide64", dict(K0=30, steps=2, new_slices=2)),
    ("tiny", dict(steps=3)),                          # J=20, R=5: generic path
    ("large", dict(K0=80, steps=2, new_slices=3, add_rows=("uniform", 1, 150))),  # interleaved big / small
    ("large", dict(K0=80, steps=2, new_slices=3, passes=2)),                      # multi-pass, fused path
    ("large", dict(K0=60, steps=2, new_slices=2, J=200)),                         # J > 128: no fused path
])
def test_fp32_mode_matches_oracle(name, kw):
    from paper_2305_18376_b200 import workloads as wl
    from paper_2305_18376_b200.stream import StreamState
    cfg = wl.scaled(wl.CONFIGS[name], **kw)
    stream = wl.make_stream(cfg)
    ps = wl.planted_state(stream)
    gpu = StreamState.from_arrays(dict(ps, passes=cfg.passes), dtype=torch.float32)
    exact = _oracle(ps, cfg.passes)
    rounded = _oracle(ps, cfg.passes)
    worst_e, worst_r = {}, {}
    for batch in stream.batches():
        res = gpu.update(batch)
        re_ = exact.update(batch)
        rr = rounded.update(_round_batch(batch))
        ids = [sid for sid, _, _ in batch.items()]
        U = np.concatenate([res.u_new[s] for s in ids])
        assert U.dtype == np.float32
        for ref, worst in ((re_, worst_e), (rr, worst_r)):
            orc_state = exact if ref is re_ else rounded
            pairs = {"U": (U, np.concatenate([ref["u_new"][s] for s in ids])),
                     "v_used": (res.v_used, ref["v_used"])}
            for nm in ("W", "C", "D", "F", "G", "V"):
                pairs[nm] = (getattr(gpu, nm), getattr(orc_state, nm))
            for k, (a, b) in pairs.items():
                worst[k] = max(worst.get(k, 0.0), rel(a, b))
    assert all(v < TOL_F32 for v in worst_e.values()), (name, worst_e)
    assert all(v < TOL_ROUNDED for v in worst_r.values()), (name, worst_r)


def test_fp32_local_error_and_pipeline():
    """local_error in the FP32 mode, and HostPipeline feeding FP32 pinned
    batches gives the same bytes as device-resident FP32 updates."""
    from paper_2305_18376_b200 import workloads as wl
    from paper_2305_18376_b200.evaluate import local_error
    from paper_2305_18376_b200.stream import HostPipeline, StreamState
    cfg = wl.scaled(wl.CONFIGS["large"], K0=200, steps=3, new_slices=3)
    stream = wl.make_stream(cfg)
    ps = wl.planted_state(stream)
    a = StreamState.from_arrays(ps, dtype=torch.float32)
    b = StreamState.from_arrays(ps, dtype=torch.float32)
    cpu = _oracle(ps, 1)
    batches = list(stream.batches())
    refs = []
    for bt in batches:
        res = a.update(bt)
        rb = _round_batch(bt)
        ref = cpu.update(rb)
        items = [(sid, rows) for sid, rows, _ in bt.items()]
        te, per = local_error(items, res.u_new, a)
        W_rows = {sid: cpu.W[cpu.row_of(sid)] for sid, _ in items}
        te_o, per_o = orc.local_error([(sid, rows) for sid, rows, _ in rb.items()], ref["u_new"], W_rows, cpu.V)
        assert abs(te - te_o) <= 1e-5 * abs(te_o)
        ids = [s for s, _ in items]
        assert rel(np.array([per[s] for s in ids]), np.array([per_o[s] for s in ids])) < 1e-5
        refs.append(np.concatenate([res.u_new[s] for s in ids]))
    Xs = [np.concatenate([r for _, r in bt.existing_rows.items()] + [ns.rows for ns in bt.new_slices])
          .astype(np.float32) for bt in batches]
    pins = [torch.as_tensor(X).pin_memory() for X in Xs]
    maxN = max(X.shape[0] for X in Xs)
    R = cfg.R
    Uh = [torch.empty((maxN, R), dtype=torch.float32).pin_memory() for _ in batches]
    pipe = HostPipeline(b, maxN, cfg.J)
    pipe.start()
    staged = pipe.put(pins[0])
    for k, bt in enumerate(batches):
        nxt = pipe.put(pins[k + 1]) if k + 1 < len(batches) else None
        ex = list(bt.existing_rows.items())
        counts = np.array([r.shape[0] for _, r in ex] + [ns.rows.shape[0] for ns in bt.new_slices])
        rows = np.array([b.row_of(s) for s, _ in ex], dtype=np.int32)
        pipe.update(staged, counts, rows, [ns.slice_id for ns in bt.new_slices], U_host=Uh[k])
        staged = nxt
    pipe.finish()
    torch.cuda.synchronize()
    for k, U in enumerate(refs):
        assert np.array_equal(Uh[k][:U.shape[0]].numpy(), U), k
    for nm in ("W", "C", "D", "F", "G", "V"):
        assert np.array_equal(getattr(a, nm), getattr(b, nm)), nm


def test_fp32_rejects_fp64_batch():
    from paper_2305_18376_b200 import workloads as wl
    from paper_2305_18376_b200.stream import StreamState
    cfg = wl.scaled(wl.CONFIGS["tiny"], K0=8, steps=1)
    stream = wl.make_stream(cfg)
    st = StreamState.from_arrays(wl.planted_state(stream), dtype=torch.float32)
    X = torch.zeros((3, cfg.J), dtype=torch.float64, device="cuda")
    with pytest.raises(TypeError):
        st.update_packed(X, np.array([3]), np.array([0], dtype=np.int32), [])


@pytest.mark.parametrize("name,kw", [
    ("wide10", dict(K0=40, steps=2, new_slices=2)),            # J = 1,024: k_row_err_mma_wide on float X / U
    ("wide64", dict(K0=24, steps=1, new_slices=2, J=520)),     # R = 64, 5 column chunks of 128, the last one short
])
def test_fp32_local_error_at_wide_j(name, kw):
    """local_error in the FP32 data mode where V does not fit in shared memory (chunked DMMA kernel)."""
    from paper_2305_18376_b200 import workloads as wl
    from paper_2305_18376_b200.evaluate import local_error
    from paper_2305_18376_b200.stream import StreamState
    cfg = wl.scaled(wl.CONFIGS[name], **kw)
    stream = wl.make_stream(cfg)
    ps = wl.planted_state(stream)
    gpu = StreamState.from_arrays(ps, dtype=torch.float32)
    cpu = _oracle(ps, 1)
    for bt in stream.batches():
        res = gpu.update(bt)
        rb = _round_batch(bt)
        ref = cpu.update(rb)
        items = [(sid, rows) for sid, rows, _ in bt.items()]
        te, per = local_error(items, res.u_new, gpu)
        W_rows = {sid: cpu.W[cpu.row_of(sid)] for sid, _ in items}
        te_o, per_o = orc.local_error([(sid, rows) for sid, rows, _ in rb.items()], ref["u_new"], W_rows, cpu.V)
        assert abs(te - te_o) <= TOL_ROUNDED * abs(te_o)
        ids = [s for s, _ in items]
        assert rel(np.array([per[s] for s in ids]), np.array([per_o[s] for s in ids])) < TOL_ROUNDED
