"""GPU parafac2_als / initialize against the reference's golden ALS vectors."""
import numpy as np
import pytest
import torch

from golden_io import batches_from, load, rel

TOL = 1e-8


def tiny_tensor(g):
    from paper_2305_18376_b200.tensor import IrregularTensor, SliceMatrix
    ids = [str(s) for s in g["init_ids"]]
    offs = np.concatenate([[0], np.cumsum(g["init_counts"])])
    return IrregularTensor(SliceMatrix(s, g["init_X"][offs[k]:offs[k + 1]]) for k, s in enumerate(ids)), ids, offs


def test_rank_and_iters_validation_on_cpu():
    from paper_2305_18376_b200.als import parafac2_als
    g = load("tiny_stream.npz")
    t, _, _ = tiny_tensor(g)
    with pytest.raises(ValueError):
        parafac2_als(t, 21, iters=2)
    with pytest.raises(ValueError):
        parafac2_als(t, 2, iters=0)


@pytest.mark.gpu
def test_parafac2_als_matches_reference_golden():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    from paper_2305_18376_b200.als import parafac2_als
    g = load("tiny_stream.npz")
    t, ids, offs = tiny_tensor(g)
    fs, info = parafac2_als(t, int(g["R"]), iters=10, seed=0, return_info=True)
    np.testing.assert_allclose(info.losses, g["als_losses"], rtol=TOL, atol=0)
    assert rel(np.concatenate([info.projections[s] for s in ids]), g["als_Q"]) < TOL
    assert rel(np.concatenate([fs.U[s] for s in ids]), g["als_U"]) < TOL
    assert rel(fs.W, g["als_W"]) < TOL and rel(fs.V, g["als_V"]) < TOL
    # fixed-sweep mode used by the refit baseline (tol=0, evaluate.py:219-221)
    f0, i0 = parafac2_als(t, int(g["R"]), iters=4, seed=7, tol=0.0, return_info=True)
    np.testing.assert_allclose(i0.losses, g["als_tol0_losses"], rtol=TOL, atol=0)
    assert rel(f0.V, g["als_tol0_V"]) < TOL and rel(f0.W, g["als_tol0_W"]) < TOL
    for s in ids[:10]:
        q = info.projections[s]
        assert np.abs(q.T @ q - np.eye(q.shape[1])).max() < 1e-10


@pytest.mark.gpu
def test_initialize_then_stream_matches_reference_golden():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    from paper_2305_18376_b200.stream import initialize
    g = load("tiny_stream.npz")
    t, ids, offs = tiny_tensor(g)
    state, info = initialize(t, int(g["R"]), iters=10, seed=0, forgetting=float(g["forgetting"]))
    for name, key in (("C", "init_C"), ("D", "init_D"), ("F", "init_F"), ("G", "init_G"),
                      ("W", "als_W"), ("V", "als_V")):
        assert rel(getattr(state, name), g[key]) < TOL, name
    assert rel(state.u_matrix(ids[3]), g["als_U"][offs[3]:offs[4]]) < TOL
    for tt, batch in enumerate(batches_from(g)):
        res = state.update(batch)
        U = np.concatenate([res.u_new[s] for s, _, _ in batch.items()])
        assert rel(U, g[f"u{tt}_U"]) < TOL
        for name in ("W", "C", "D", "F", "G", "V"):
            assert rel(getattr(state, name), g[f"u{tt}_{name}"]) < TOL, (tt, name)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["medium", "daily"])
def test_parafac2_als_matches_reference_at_baseline_shapes(name):
    """parafac2_als at the medium (K=1,000) and daily (K=4,700) BASELINE shapes
    against the reference's own fit of the same seeded tensor
    (tests/golden/make_golden_als.py): loss log, W, V, every slice's
    ||U_k||_F, U_k / Q_k of the first slices; early-exit mode (tol=1e-8) and
    the refit baseline's fixed-sweep mode (tol=0, evaluate.py:219-221)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    from paper_2305_18376_b200 import workloads as wl
    from paper_2305_18376_b200.als import parafac2_als
    g = load(f"als_{name}.npz")
    cfg = wl.CONFIGS[name]
    t = wl.make_stream(cfg, exact=False).initial_tensor()
    ids = t.slice_ids
    fs, info = parafac2_als(t, int(g["R"]), iters=10, seed=0, return_info=True)
    assert len(info.losses) == len(g["losses"])
    np.testing.assert_allclose(info.losses, g["losses"], rtol=TOL, atol=0)
    assert rel(fs.W, g["W"]) < TOL and rel(fs.V, g["V"]) < TOL
    assert rel(np.array([np.linalg.norm(fs.U[s]) for s in ids]), g["U_norms"]) < TOL
    for k in range(8):
        assert rel(fs.U[ids[k]], g[f"U{k}"]) < TOL, k
        assert rel(info.projections[ids[k]], g[f"Q{k}"]) < TOL, k
    f0, i0 = parafac2_als(t, int(g["R"]), iters=4, seed=7, tol=0.0, return_info=True)
    assert len(i0.losses) == 4
    np.testing.assert_allclose(i0.losses, g["tol0_losses"], rtol=TOL, atol=0)
    assert rel(f0.W, g["tol0_W"]) < TOL and rel(f0.V, g["tol0_V"]) < TOL
