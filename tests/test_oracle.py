"""Pin the CPU oracle (oracle/) to the reference's own outputs.

The golden vectors were produced by running the reference p2stream package
(tests/golden/make_golden.py).  If /root/reference is present the live
reference is also compared directly.
"""
import os
import sys
from pathlib import Path

import numpy as np
import pytest

from golden_io import batches_from, load, planted_arrays, rel
from oracle import dash_oracle as orc

TOL = 1e-12   # oracle vs reference: same algorithm, same arithmetic order


def run_oracle_stream(g, prefix, state, check_every=True):
    for t, batch in enumerate(batches_from(g, prefix)):
        res = orc.OracleStreamState.update(state, batch)
        ids = [sid for sid, _, _ in batch.items()]
        U = np.concatenate([res["u_new"][sid] for sid in ids])
        assert rel(U, g[f"{prefix}u{t}_U"]) < TOL
        for name in ("W", "C", "D", "F", "G", "V"):
            assert rel(getattr(state, name), g[f"{prefix}u{t}_{name}"]) < TOL, (t, name)
        assert rel(res["v_used"], g[f"{prefix}u{t}_v_used"]) < TOL
        assert state.slice_ids == [str(s) for s in g[f"{prefix}u{t}_slice_ids"]]
        items = [(sid, rows) for sid, rows, _ in batch.items()]
        wrows = {sid: state.W[state.row_of(sid)] for sid in ids}
        te, per = orc.local_error(items, res["u_new"], wrows, state.V)
        assert abs(te - float(g[f"{prefix}u{t}_local_error"])) <= TOL * abs(te)
    return state


def planted_oracle(g, prefix, passes=1, use_kernel=True):
    p = planted_arrays(g, prefix)
    R = p["V"].shape[1]
    return orc.OracleStreamState(
        p["slice_ids"], {sid: [np.zeros((0, R))] for sid in p["slice_ids"]},
        p["W"], p["V"], p["C"], p["D"], p["F"], p["G"], p["forgetting"],
        passes=passes, use_kernel=use_kernel)


def test_c_kernel_bit_exact_vs_numba_golden():
    g = load("kernel.npz")
    for n in range(int(g["n_cases"])):
        got = orc.group_update(g[f"k{n}_xv"], g[f"k{n}_vtv"], g[f"k{n}_s"], g[f"k{n}_c_old"],
                               g[f"k{n}_d_old"], float(g[f"k{n}_lam"]), 1e-10)
        for key, val in zip(("u", "us", "c_new", "d_new", "w", "g_fresh"), got[:6]):
            ref = g[f"k{n}_out_{key}"]
            assert np.array_equal(val, ref) or rel(val, ref) < 1e-15, (n, key)
        assert got[6] == bool(g[f"k{n}_out_ok"])


def test_tiny_stream_als_init_and_updates():
    g = load("tiny_stream.npz")
    ids = [str(s) for s in g["init_ids"]]
    counts = g["init_counts"]
    offs = np.concatenate([[0], np.cumsum(counts)])
    slices = [(sid, g["init_X"][offs[k]:offs[k + 1]]) for k, sid in enumerate(ids)]
    R = int(g["R"])
    U, W, V, losses, proj, H = orc.parafac2_als(slices, R, iters=10, seed=0)
    assert np.allclose(losses, g["als_losses"], rtol=1e-10, atol=0)
    assert rel(np.concatenate([proj[s] for s in ids]), g["als_Q"]) < 1e-9
    assert rel(np.concatenate([U[s] for s in ids]), g["als_U"]) < 1e-9
    assert rel(W, g["als_W"]) < 1e-9 and rel(V, g["als_V"]) < 1e-9
    c, D, F, G = orc.init_helpers(slices, U, W, V)
    assert rel(np.stack([c[s] for s in ids]), g["init_C"]) < 1e-9
    assert rel(np.stack([D[s] for s in ids]), g["init_D"]) < 1e-9
    assert rel(F, g["init_F"]) < 1e-9 and rel(G, g["init_G"]) < 1e-9
    # ALS in fixed-sweep mode (tol=0)
    _, W0, V0, l0, _, _ = orc.parafac2_als(slices, R, iters=4, seed=7, tol=0.0)
    assert np.allclose(l0, g["als_tol0_losses"], rtol=1e-10, atol=0)
    assert rel(V0, g["als_tol0_V"]) < 1e-9
    # updates start from the reference's own initial state (bit-identical inputs)
    state = orc.OracleStreamState(
        ids, {s: [g["als_U"][offs[k]:offs[k + 1]]] for k, s in enumerate(ids)},
        g["als_W"], g["als_V"], g["init_C"], g["init_D"], g["init_F"], g["init_G"],
        float(g["forgetting"]))
    run_oracle_stream(g, "", state)


@pytest.mark.parametrize("tag,fast", [("fast_", True), ("numpy_", False)])
def test_multipass_both_reference_paths(tag, fast):
    g = load("multipass.npz")
    state = planted_oracle(g, tag, passes=int(g[f"{tag}passes"]), use_kernel=fast)
    run_oracle_stream(g, tag, state)


@pytest.mark.parametrize("prefix", ["a_", "b_", "c_"])
def test_edge_streams(prefix):
    g = load("edge.npz")
    state = planted_oracle(g, prefix)
    run_oracle_stream(g, prefix, state)


def test_known_answers():
    # scalar S-row case from the reference's own test (test_stream_ops.py:150-153)
    v = np.array([[1.0], [2.0]])
    w = orc.ridge_solve((v.T @ v) * np.array([[2.0]]), np.array([10.0]))
    assert w[0] == pytest.approx(1.0, rel=1e-9)
    with pytest.raises(orc.OracleSolveError):
        orc.ridge_solve(np.zeros((2, 2)), np.ones((2, 4)))


REF = Path("/root/reference/pkg/src")


@pytest.mark.skipif(not REF.exists(), reason="reference not present (GPU box)")
def test_oracle_matches_live_reference_medium_shape():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, str(REF))
    import p2stream
    from paper_2305_18376_b200 import workloads as wl
    cfg = wl.scaled(wl.CONFIGS["medium"], K0=30, steps=3)
    stream = wl.make_stream(cfg)
    ps = wl.planted_state(stream)
    R = cfg.R
    ref = p2stream.StreamState(list(ps["slice_ids"]), {s: [np.zeros((0, R))] for s in ps["slice_ids"]},
                               ps["W"].copy(), ps["V"].copy(), ps["C"].copy(), ps["D"].copy(),
                               ps["F"].copy(), ps["G"].copy(), ps["forgetting"])
    me = orc.OracleStreamState(list(ps["slice_ids"]), {s: [np.zeros((0, R))] for s in ps["slice_ids"]},
                               ps["W"], ps["V"], ps["C"], ps["D"], ps["F"], ps["G"], ps["forgetting"])
    for b in stream.batches():
        rb = p2stream.UpdateBatch(b.update_index, dict(b.existing_rows),
                                  [p2stream.NewSlice(n.slice_id, n.rows, 0) for n in b.new_slices], (0, 0))
        ref.update(rb)
        me.update(b)
        for name in ("W", "C", "D", "F", "G", "V"):
            assert rel(getattr(me, name), getattr(ref, name)) < 1e-12
