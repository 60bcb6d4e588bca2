"""Checkpoints (reference stream.py:409-540) and ingest normalisation
(reference tensor.py:252-360), pinned to files / outputs the reference itself
wrote (tests/golden/make_golden.py: ckpt_ref.json, ckpt_ref.npz, ckpt.npz).

CPU tests: normalisation is bit-exact against the reference's normalize_batch
chain, and save_state reproduces the reference's checkpoint bytes / arrays for
the same state.  GPU tests: load_state of the reference's files resumes the
stream on the device and follows the reference's trajectory (1e-8).
"""
import json

import numpy as np
import pytest

from golden_io import GOLDEN, batch_from, batches_from, load, rel
from paper_2305_18376_b200.checkpoint import STATE_FORMAT_VERSION, load_state, save_state
from paper_2305_18376_b200.tensor import (CAUSAL, GLOBAL, ColumnStats, DatasetError, IrregularTensor, NewSlice,
                                          SliceMatrix, UpdateBatch, global_stats, normalize_batch,
                                          normalize_tensor)

TOL = 1e-8


class HostState:
    """Host stand-in with the StreamState attributes save_state reads."""

    def __init__(self, doc):
        self.slice_ids = list(doc["slice_ids"])
        self._u = {sid: np.asarray(doc["u"][sid], dtype=float) for sid in self.slice_ids}
        self.W = np.asarray(doc["w"], dtype=float)
        self.V = np.asarray(doc["v"], dtype=float)
        self.C = np.asarray([doc["helpers"]["c"][s] for s in self.slice_ids], dtype=float)
        self.D = np.asarray([doc["helpers"]["d"][s] for s in self.slice_ids], dtype=float)
        self.F = np.asarray(doc["helpers"]["f"], dtype=float)
        self.G = np.asarray(doc["helpers"]["g"], dtype=float)
        self.forgetting, self.update_index = doc["forgetting"], doc["update_index"]
        self.passes, self.rank = doc["passes"], doc["rank"]

    def u_matrix(self, sid):
        return self._u[sid].copy()


def _ref_stats(doc):
    raw = doc["column_stats"]
    return ColumnStats({k: np.asarray(v, dtype=float) for k, v in raw["minimum"].items()},
                       {k: np.asarray(v, dtype=float) for k, v in raw["maximum"].items()})


def test_normalize_batch_chain_matches_reference_bitwise():
    g = load("ckpt.npz")
    # the reference chain starts from global_stats of the tiny initial tensor
    from paper_2305_18376_b200 import workloads as wl
    init = wl.make_stream("tiny").initial_tensor()
    stats = global_stats(IrregularTensor(SliceMatrix(s.slice_id, s.rows) for s in init.slices))
    for t in range(int(g["n_norm"])):
        b = batch_from(g, "n", t)
        nb, stats = normalize_batch(b, stats)
        Xn = np.concatenate([nb.existing_rows[s] for s in nb.existing_rows] + [ns.rows for ns in nb.new_slices])
        assert np.array_equal(Xn, g[f"nb{t}_Xn"]), t
    ids = [str(s) for s in g["nstats_ids"]]
    assert sorted(stats.minimum) == ids
    assert np.array_equal(np.stack([stats.minimum[s] for s in ids]), g["nstats_min"])
    assert np.array_equal(np.stack([stats.maximum[s] for s in ids]), g["nstats_max"])


def test_normalize_policies_and_errors():
    rows = np.array([[1.0, 5.0, 2.0], [3.0, 5.0, 4.0]])
    t, st = normalize_tensor(IrregularTensor([SliceMatrix("a", rows)]))
    assert np.array_equal(t.slices[0].rows, [[0.0, 0.0, 0.0], [1.0, 0.0, 1.0]])  # zero-width column -> 0
    assert np.array_equal(st.minimum["a"], [1.0, 5.0, 2.0])
    b = UpdateBatch(1, {"a": np.array([[5.0, 5.0, 6.0]])}, [NewSlice("n", rows, 1)], (1, 1))
    nb, st2 = normalize_batch(b, st, GLOBAL)
    assert np.array_equal(nb.existing_rows["a"], [[2.0, 0.0, 2.0]])
    assert not st2.has("n") and np.array_equal(st2.maximum["a"], st.maximum["a"])
    nb, st3 = normalize_batch(b, st, CAUSAL)
    assert st3.has("n") and np.array_equal(st3.maximum["a"], [5.0, 5.0, 6.0])
    with pytest.raises(DatasetError):
        normalize_batch(UpdateBatch(1, {"zz": rows}, [], (1, 1)), st)
    with pytest.raises(ValueError):
        normalize_batch(b, st, "sometimes")


def test_save_state_json_reproduces_reference_bytes(tmp_path):
    ref = (GOLDEN / "ckpt_ref.json").read_text()
    doc = json.loads(ref)
    assert doc["format_version"] == STATE_FORMAT_VERSION
    out = tmp_path / "s.json"
    save_state(HostState(doc), out, column_stats=_ref_stats(doc))
    assert out.read_text() == ref


def test_save_state_npz_matches_reference_arrays(tmp_path):
    doc = json.loads((GOLDEN / "ckpt_ref.json").read_text())
    out = tmp_path / "s.npz"
    save_state(HostState(doc), out, column_stats=_ref_stats(doc))
    with np.load(GOLDEN / "ckpt_ref.npz") as want, np.load(out) as got:
        assert sorted(want.files) == sorted(got.files)
        for k in want.files:
            if k == "meta":
                assert json.loads(bytes(got[k]).decode()) == json.loads(bytes(want[k]).decode())
            else:
                assert np.array_equal(got[k], want[k]), k


def test_bad_suffix_and_version(tmp_path):
    doc = json.loads((GOLDEN / "ckpt_ref.json").read_text())
    with pytest.raises(ValueError, match="suffix"):
        save_state(HostState(doc), tmp_path / "s.pkl")
    with pytest.raises(ValueError, match="suffix"):
        load_state(tmp_path / "s.pkl")
    doc["format_version"] = 99
    p = tmp_path / "v.json"
    p.write_text(json.dumps(doc))
    with pytest.raises(ValueError, match="format"):
        load_state(p)


@pytest.mark.gpu
@pytest.mark.parametrize("suffix", [".json", ".npz"])
def test_resume_from_reference_checkpoint_on_gpu(suffix, tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    g = load("ckpt.npz")
    state, stats = load_state(GOLDEN / f"ckpt_ref{suffix}")
    doc = json.loads((GOLDEN / "ckpt_ref.json").read_text())
    assert state.update_index == doc["update_index"] and state.slice_ids == doc["slice_ids"]
    assert sorted(stats.minimum) == sorted(doc["column_stats"]["minimum"])
    # a loaded GPU state writes the reference's bytes back
    out = tmp_path / "again.json"
    save_state(state, out, column_stats=stats)
    assert out.read_text() == (GOLDEN / "ckpt_ref.json").read_text()
    for t, batch in enumerate(batches_from(g, "r")):
        res = state.update(batch)
        ids = [sid for sid, _, _ in batch.items()]
        U = np.concatenate([res.u_new[s] for s in ids])
        assert rel(U, g[f"ru{t}_U"]) < TOL
        for name in ("W", "C", "D", "F", "G", "V"):
            assert rel(getattr(state, name), g[f"ru{t}_{name}"]) < TOL, (t, name)
    assert state.update_index == doc["update_index"] + int(g["rn_updates"])


@pytest.mark.gpu
def test_host_pipeline_updates_keep_u_history_for_save_state(tmp_path):
    """update_packed / HostPipeline record the U history like update()
    (reference stream.py:352-360): after serving the reference checkpoint's
    follow-up batches through HostPipeline, save_state writes the same bytes
    as the dict-path StreamState.update run, and every slice's U history is
    its checkpointed block plus the reference's u_new rows."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_18376_b200.stream import HostPipeline
    g = load("ckpt.npz")
    a, stats = load_state(GOLDEN / "ckpt_ref.json")
    b, _ = load_state(GOLDEN / "ckpt_ref.json")
    u0 = {sid: a.u_matrix(sid) for sid in a.slice_ids}
    batches = list(batches_from(g, "r"))
    for bt in batches:
        a.update(bt)
    Xs, metas = [], []
    for bt in batches:
        ex = list(bt.existing_rows.items())
        Xs.append(np.concatenate([r for _, r in ex] + [ns.rows for ns in bt.new_slices]))
        metas.append((np.array([r.shape[0] for _, r in ex] + [ns.rows.shape[0] for ns in bt.new_slices]),
                      [sid for sid, _ in ex], [ns.slice_id for ns in bt.new_slices]))
    pins = [torch.as_tensor(X).pin_memory() for X in Xs]
    pipe = HostPipeline(b, max(X.shape[0] for X in Xs), b.J)
    pipe.start()
    for k, (counts, ex_ids, new) in enumerate(metas):
        staged = pipe.put(pins[k])
        rows = np.array([b.row_of(s) for s in ex_ids], dtype=np.int32)
        pipe.update(staged, counts, rows, new)
    pipe.finish()
    torch.cuda.synchronize()
    b.check()
    pa, pb = tmp_path / "a.json", tmp_path / "b.json"
    save_state(a, pa, column_stats=stats)
    save_state(b, pb, column_stats=stats)
    assert pa.read_text() == pb.read_text()
    # U history = checkpointed block + the reference's u_new per update
    for sid in b.slice_ids:
        want = [u0[sid]] if sid in u0 else []
        for t, bt in enumerate(batches):
            ids = [s for s, _, _ in bt.items()]
            if sid in ids:
                k = ids.index(sid)
                offs = np.concatenate([[0], np.cumsum([r.shape[0] for _, r, _ in bt.items()])])
                want.append(g[f"ru{t}_U"][offs[k]:offs[k + 1]])
        got = b.u_matrix(sid)
        want = np.vstack(want)
        assert got.shape == want.shape, sid
        assert rel(got, want) < TOL, sid
    # npz round trip of the served state resumes with identical factors
    pz = tmp_path / "b.npz"
    save_state(b, pz, column_stats=stats)
    c, _ = load_state(pz)
    for name in ("W", "C", "D", "F", "G", "V"):
        assert np.array_equal(getattr(c, name), getattr(b, name)), name
