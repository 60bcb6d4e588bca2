"""GPU parity of the DASH update (CUDA path through the C ABI) against the
reference's golden vectors and the CPU oracle.

Tolerance (north_star): factors and fitness within 1e-8 normwise relative
(max|a-b| / max|b|) in FP64.
"""
import numpy as np
import pytest
import torch

from golden_io import batches_from, load, planted_arrays, rel
from oracle import dash_oracle as orc

pytestmark = pytest.mark.gpu

TOL = 1e-8


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_18376_b200.build import build_library
    build_library()


def gpu_state_from_planted(p, passes=1):
    from paper_2305_18376_b200.stream import StreamState
    return StreamState.from_arrays(dict(p, passes=passes))


def oracle_from_planted(p, passes=1):
    R = p["V"].shape[1]
    return orc.OracleStreamState(p["slice_ids"], {s: [np.zeros((0, R))] for s in p["slice_ids"]},
                                 p["W"], p["V"], p["C"], p["D"], p["F"], p["G"],
                                 p["forgetting"], passes=passes)


def compare_update(t, state, res, g, prefix, batch):
    ids = [sid for sid, _, _ in batch.items()]
    U = np.concatenate([res.u_new[sid] for sid in ids])
    errs = {"U": rel(U, g[f"{prefix}u{t}_U"])}
    for name in ("W", "C", "D", "F", "G", "V"):
        errs[name] = rel(getattr(state, name), g[f"{prefix}u{t}_{name}"])
    errs["v_used"] = rel(res.v_used, g[f"{prefix}u{t}_v_used"])
    bad = {k: v for k, v in errs.items() if not v < TOL}
    assert not bad, (t, bad)
    assert state.slice_ids == [str(s) for s in g[f"{prefix}u{t}_slice_ids"]]
    return errs


def test_group_update_seam_matches_numba_golden():
    from paper_2305_18376_b200.kernels import group_update
    g = load("kernel.npz")
    for n in range(int(g["n_cases"])):
        got = group_update(g[f"k{n}_xv"], g[f"k{n}_vtv"], g[f"k{n}_s"], g[f"k{n}_c_old"],
                           g[f"k{n}_d_old"], float(g[f"k{n}_lam"]), 1e-10)
        for key, val in zip(("u", "us", "c_new", "d_new", "w", "g_fresh"), got[:6]):
            assert rel(val, g[f"k{n}_out_{key}"]) < 1e-10, (n, key)
        assert got[6] == bool(g[f"k{n}_out_ok"])


def test_tiny_stream_matches_reference_golden():
    from paper_2305_18376_b200.stream import StreamState
    g = load("tiny_stream.npz")
    ids = [str(s) for s in g["init_ids"]]
    offs = np.concatenate([[0], np.cumsum(g["init_counts"])])
    state = StreamState(ids, {s: [g["als_U"][offs[k]:offs[k + 1]]] for k, s in enumerate(ids)},
                        g["als_W"], g["als_V"], g["init_C"], g["init_D"], g["init_F"],
                        g["init_G"], float(g["forgetting"]))
    for t, batch in enumerate(batches_from(g)):
        res = state.update(batch)
        compare_update(t, state, res, g, "", batch)
        assert res.update_index == t + 1
    # U history: initial block + every appended block, in order
    for k, sid in enumerate(ids[:5]):
        U = state.u_matrix(sid)
        assert U.shape[0] == g["init_counts"][k] + sum(
            int(g[f"b{t}_counts"][list(map(str, g[f"b{t}_ids"])).index(sid)])
            for t in range(int(g["n_updates"])) if sid in set(map(str, g[f"b{t}_ids"])))


@pytest.mark.parametrize("tag", ["fast_", "numpy_"])
def test_multipass_matches_golden(tag):
    g = load("multipass.npz")
    state = gpu_state_from_planted(planted_arrays(g, tag), passes=int(g[f"{tag}passes"]))
    for t, batch in enumerate(batches_from(g, tag)):
        res = state.update(batch)
        compare_update(t, state, res, g, tag, batch)


@pytest.mark.parametrize("prefix", ["a_", "b_", "c_"])
def test_edge_streams_match_golden(prefix):
    g = load("edge.npz")
    state = gpu_state_from_planted(planted_arrays(g, prefix))
    for t, batch in enumerate(batches_from(g, prefix)):
        res = state.update(batch)
        compare_update(t, state, res, g, prefix, batch)


def stream_parity(cfg, steps_check=None):
    from paper_2305_18376_b200 import workloads as wl
    stream = wl.make_stream(cfg)
    ps = wl.planted_state(stream)
    gpu = gpu_state_from_planted(ps, passes=cfg.passes)
    cpu = oracle_from_planted(ps, passes=cfg.passes)
    worst = {}
    for batch in stream.batches():
        res = gpu.update(batch)
        ref = cpu.update(batch)
        ids = [sid for sid, _, _ in batch.items()]
        pairs = {"U": (np.concatenate([res.u_new[s] for s in ids]),
                       np.concatenate([ref["u_new"][s] for s in ids])),
                 "v_used": (res.v_used, ref["v_used"])}
        for name in ("W", "C", "D", "F", "G", "V"):
            pairs[name] = (getattr(gpu, name), getattr(cpu, name))
        for k, (a, b) in pairs.items():
            worst[k] = max(worst.get(k, 0.0), rel(a, b))
    bad = {k: v for k, v in worst.items() if not v < TOL}
    assert not bad, (cfg.name, worst)
    return worst


@pytest.mark.parametrize("name,kw", [
    ("medium", dict(K0=150, steps=3)),
    ("daily", dict(K0=300, steps=6)),
    ("large", dict(K0=120, steps=2, new_slices=3)),
    ("wide10", dict(K0=40, steps=2, new_slices=2)),
    ("wide32", dict(K0=40, steps=2, new_slices=2)),
    ("wide64", dict(K0=30, steps=2, new_slices=2)),
])
def test_config_shaped_streams_match_oracle(name, kw):
    from paper_2305_18376_b200 import workloads as wl
    cfg = wl.scaled(wl.CONFIGS[name], **kw)
    stream_parity(cfg)


@pytest.mark.parametrize("name,kw", [
    # existing slices of 1..150 rows: big and small slices interleave, so tiles on
    # both sides of a big slice are shared with small ones (boundary U o w zeroing)
    ("large", dict(K0=80, steps=2, new_slices=3, add_rows=("uniform", 1, 150))),
    ("large", dict(K0=80, steps=2, new_slices=3, passes=2)),      # multi-pass on the fused path
    ("large", dict(K0=60, steps=2, new_slices=2, R=14)),          # R < 16, even: fused path
    ("large", dict(K0=60, steps=2, new_slices=2, R=13)),          # odd R: k_xv2 / k_slices2 path
    ("medium", dict(K0=100, steps=2, J=120)),                     # J < 128 in 8 box strips
    ("large", dict(K0=60, steps=2, new_slices=2, J=200)),         # J > 128: TMA GEMMs + k_big (no fused path)
])
def test_fused_path_edges_match_oracle(name, kw):
    from paper_2305_18376_b200 import _native as nat
    from paper_2305_18376_b200 import workloads as wl
    cfg = wl.scaled(wl.CONFIGS[name], **kw)
    stream_parity(cfg)
    if cfg.R % 2 == 0 and cfg.J <= 128:  # the fused big-slice path ran
        stream = wl.make_stream(cfg)
        st = gpu_state_from_planted(wl.planted_state(stream), passes=cfg.passes)
        st.update(next(stream.batches()))
        assert nat.lib().dash_ctx_path_flags(st._ctx) & nat.PATH_BIGX


def _spread_weights(ps):
    """W rows with entries over many magnitudes (and signs, and exact zeros):
    the small-slice kernel's A system S (vtv + sh S^-2) S takes its Neumann
    fast path for most slices, the second-order term matters for the 1e-3 ..
    1e-2 entries, and the exact sweep runs for the tiny / zero ones."""
    W = ps["W"].copy()
    K, R = W.shape
    rng = np.random.default_rng(7)
    scales = np.array([1.0, 1e-2, 3e-3, -2e-3, 1e-4, 1e-6, 0.0])
    for k in range(K):
        if k % 3 == 0:
            cols = rng.choice(R, size=2, replace=False)
            W[k, cols] *= scales[rng.integers(len(scales), size=2)]
    return dict(ps, W=W)


@pytest.mark.parametrize("R", [16, 10])
def test_small_slice_neumann_and_sweep_paths_match_oracle(R):
    from paper_2305_18376_b200 import workloads as wl
    cfg = wl.scaled(wl.CONFIGS["large"], K0=150, steps=2, new_slices=2, R=R)
    stream = wl.make_stream(cfg)
    ps = _spread_weights(wl.planted_state(stream))
    gpu = gpu_state_from_planted(ps)
    cpu = oracle_from_planted(ps)
    for batch in stream.batches():
        res = gpu.update(batch)
        ref = cpu.update(batch)
        ids = [sid for sid, _, _ in batch.items()]
        errs = {"U": rel(np.concatenate([res.u_new[s] for s in ids]),
                         np.concatenate([ref["u_new"][s] for s in ids]))}
        for name in ("W", "C", "D", "F", "G", "V"):
            errs[name] = rel(getattr(gpu, name), getattr(cpu, name))
        bad = {k: v for k, v in errs.items() if not v < TOL}
        assert not bad, errs


def test_update_is_bit_reproducible():
    from paper_2305_18376_b200 import workloads as wl
    cfg = wl.scaled(wl.CONFIGS["large"], K0=100, steps=2, new_slices=2)
    outs = []
    for _ in range(2):
        stream = wl.make_stream(cfg)
        st = gpu_state_from_planted(wl.planted_state(stream))
        for b in stream.batches():
            st.update(b)
        outs.append((st.V.copy(), st.W.copy(), st.C.copy(), st.D.copy(), st.F.copy(), st.G.copy()))
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


def test_dormant_slices_untouched_and_unknown_ids_rejected():
    from paper_2305_18376_b200 import workloads as wl
    from paper_2305_18376_b200.tensor import NewSlice, UpdateBatch
    cfg = wl.scaled(wl.CONFIGS["tiny"], K0=8, steps=1)
    stream = wl.make_stream(cfg)
    st = gpu_state_from_planted(wl.planted_state(stream))
    batch = next(stream.batches())
    dormant = "s000000"
    trimmed = UpdateBatch(1, {k: v for k, v in batch.existing_rows.items() if k != dormant},
                          batch.new_slices, (1, 1))
    row = st.row_of(dormant)
    before = (st.W[row].copy(), st.C[row].copy(), st.D[row].copy())
    st.update(trimmed)
    assert np.array_equal(st.W[row], before[0])
    assert np.array_equal(st.C[row], before[1])
    assert np.array_equal(st.D[row], before[2])
    with pytest.raises(ValueError, match="ghost"):
        st.update(UpdateBatch(2, {"ghost": np.ones((2, cfg.J))}, [], (2, 2)))
    with pytest.raises(ValueError, match="as new"):
        st.update(UpdateBatch(2, {}, [NewSlice(dormant, np.ones((2, cfg.J)), 2)], (2, 2)))


def test_singular_system_raises_solve_error_naming_slice():
    from paper_2305_18376_b200 import workloads as wl
    from paper_2305_18376_b200.linalg import SolveError
    cfg = wl.scaled(wl.CONFIGS["tiny"], K0=6, steps=1)
    stream = wl.make_stream(cfg)
    ps = wl.planted_state(stream)
    ps["W"][2] = 0.0      # s = 0 -> A = 0 (+ zero ridge): singular
    st = gpu_state_from_planted(ps)
    batch = next(stream.batches())
    with pytest.raises(SolveError) as ei:
        st.update(batch)
    assert ei.value.slice_id == "s000002"


def test_local_error_matches_golden():
    from paper_2305_18376_b200.evaluate import local_error
    g = load("edge.npz")
    state = gpu_state_from_planted(planted_arrays(g, "a_"))
    for t, batch in enumerate(batches_from(g, "a_")):
        res = state.update(batch)
        items = [(sid, rows) for sid, rows, _ in batch.items()]
        te, per = local_error(items, res.u_new, state)
        want = float(g[f"a_u{t}_local_error"])
        assert abs(te - want) <= TOL * abs(want)
        ids = [sid for sid, _ in items]
        assert rel(np.array([per[s] for s in ids]), g[f"a_u{t}_slice_error"]) < TOL


def test_init_helpers_matches_golden():
    from paper_2305_18376_b200.als import FactorSet
    from paper_2305_18376_b200.stream import init_helpers
    from paper_2305_18376_b200.tensor import IrregularTensor, SliceMatrix
    g = load("tiny_stream.npz")
    ids = [str(s) for s in g["init_ids"]]
    offs = np.concatenate([[0], np.cumsum(g["init_counts"])])
    tensor = IrregularTensor(SliceMatrix(s, g["init_X"][offs[k]:offs[k + 1]]) for k, s in enumerate(ids))
    fs = FactorSet(ids, {s: g["als_U"][offs[k]:offs[k + 1]] for k, s in enumerate(ids)},
                   g["als_W"], g["als_V"])
    h = init_helpers(tensor, fs, forgetting=1.0)
    assert rel(np.stack([h.c[s] for s in ids]), g["init_C"]) < TOL
    assert rel(np.stack([h.D[s] for s in ids]), g["init_D"]) < TOL
    assert rel(h.F, g["init_F"]) < TOL and rel(h.G, g["init_G"]) < TOL


def test_ridge_solve_matches_oracle():
    from paper_2305_18376_b200.kernels import ridge_solve
    rng = np.random.default_rng(5)
    for n, m in ((1, 3), (5, 7), (16, 40), (32, 3)):
        base = rng.standard_normal((4, n, n + 2))
        lhs = base @ base.transpose(0, 2, 1)
        rhs = rng.standard_normal((4, n, m))
        assert rel(ridge_solve(lhs, rhs), orc.ridge_solve(lhs, rhs)) < 1e-10


def _packed(state, batch):
    """UpdateBatch -> update_packed arguments (items() order: existing, then new)."""
    ex = list(batch.existing_rows.items())
    X = np.concatenate([r for _, r in ex] + [ns.rows for ns in batch.new_slices])
    counts = np.array([r.shape[0] for _, r in ex] + [ns.rows.shape[0] for ns in batch.new_slices])
    rows = np.array([state.row_of(s) for s, _ in ex], dtype=np.int32)
    return X, counts, rows, [ns.slice_id for ns in batch.new_slices]


def test_host_pipeline_matches_device_resident_updates():
    """HostPipeline (overlapped pinned H2D / update / D2H) is bit-identical to
    update_packed on device-resident batches."""
    from paper_2305_18376_b200 import workloads as wl
    from paper_2305_18376_b200.stream import HostPipeline
    cfg = wl.scaled(wl.CONFIGS["large"], K0=200, steps=4, new_slices=3)
    stream = wl.make_stream(cfg)
    ps = wl.planted_state(stream)
    a = gpu_state_from_planted(ps)
    b = gpu_state_from_planted(ps)
    batches = list(stream.batches())
    ref = []
    for bt in batches:
        X, counts, rows, new = _packed(a, bt)
        U, vu = a.update_packed(torch.as_tensor(X, device="cuda"), counts, rows, new)
        ref.append((U.cpu().numpy(), vu.cpu().numpy()))
    Xs = [np.concatenate([r for _, r in bt.existing_rows.items()] + [ns.rows for ns in bt.new_slices])
          for bt in batches]
    pins = [torch.as_tensor(X).pin_memory() for X in Xs]
    maxN = max(X.shape[0] for X in Xs)
    R = ps["V"].shape[1]
    Uh = [torch.empty((maxN, R), dtype=torch.float64).pin_memory() for _ in batches]
    vh = [torch.empty((cfg.J, R), dtype=torch.float64).pin_memory() for _ in batches]
    pipe = HostPipeline(b, maxN, cfg.J)
    pipe.start()
    staged = pipe.put(pins[0])
    for k, bt in enumerate(batches):
        nxt = pipe.put(pins[k + 1]) if k + 1 < len(batches) else None
        _, counts, rows, new = _packed(b, bt)  # state rows: after the previous update registered its slices
        pipe.update(staged, counts, rows, new, U_host=Uh[k], v_host=vh[k])
        staged = nxt
    pipe.finish()
    torch.cuda.synchronize()
    for k, (U, vu) in enumerate(ref):
        assert np.array_equal(Uh[k][:U.shape[0]].numpy(), U), k
        assert np.array_equal(vh[k].numpy(), vu), k
    for name in ("W", "C", "D", "F", "G", "V"):
        assert np.array_equal(getattr(a, name), getattr(b, name)), name


@pytest.mark.parametrize("name", ["large", "wide32", "wide64"])
def test_indefinite_G_takes_the_lu_path_like_the_reference(name):
    """G0 = -10 I makes lam G0 + g indefinite: every pivot test of the V
    solve (the sweep at R <= 16; the tile Cholesky of k_vsolvew at R = 32 / 64,
    which then hands the launch to the sweep / LU kernel behind it) fails and
    the LU fallback (the reference's np.linalg.solve, linalg.py:25-45) must
    give the reference's V."""
    from paper_2305_18376_b200 import _native as nat
    from paper_2305_18376_b200 import workloads as wl
    cfg = wl.scaled(wl.CONFIGS[name], K0=40, steps=1, new_slices=2)
    stream = wl.make_stream(cfg)
    ps = wl.planted_state(stream)
    ps["G"] = -10.0 * np.eye(cfg.R) * np.abs(ps["G"]).max()
    gpu = gpu_state_from_planted(ps)
    cpu = oracle_from_planted(ps)
    nat.lib().dash_ctx_fallbacks(gpu._ctx, nat.stream_ptr(), 1)
    batch = next(stream.batches())
    gpu.update(batch)
    cpu.update(batch)
    for name in ("V", "F", "G", "W"):
        assert rel(getattr(gpu, name), getattr(cpu, name)) < TOL, name
    assert nat.lib().dash_ctx_fallbacks(gpu._ctx, nat.stream_ptr(), 1) >= 1


@pytest.mark.parametrize("name,kw", [
    ("wide10", dict(K0=40, steps=2, new_slices=2, J=130)),             # just past the J <= 128 tensor-map path
    ("wide10", dict(K0=40, steps=2, new_slices=2, J=257, R=16)),       # two column blocks, the second one column wide
    ("wide10", dict(K0=30, steps=2, new_slices=2, J=1000, R=6)),       # J not a multiple of 16 / 64; R bucket 8
    ("wide32", dict(K0=30, steps=2, new_slices=2, J=600, R=30)),       # R < 32: padded ranks in k_xvw / k_fgemmw / k_slicesw
    ("wide64", dict(K0=24, steps=2, new_slices=2, J=1030, R=50)),      # 9 column blocks of 128, G tiles over 9 x 8 warps
    ("wide64", dict(K0=24, steps=2, new_slices=2, J=300)),             # 3 column blocks: too few warps for the G tiles -> generic GEMMs
    ("wide32", dict(K0=30, steps=2, new_slices=2, passes=2)),          # multi-pass: US / G recomputed per pass
    ("wide10", dict(K0=1, steps=2, new_slices=0, add_rows=("fixed", 1))),  # one slice, one row per update
    ("wide10", dict(K0=40, steps=2, new_slices=2, R=9)),               # odd R: generic register-staged GEMMs
])
def test_wide_j_path_edges_match_oracle(name, kw):
    """The wide-J tensor-map GEMMs (dash_widej.cuh), k_us_rows and the wide row-error kernel at the
    edges of their tilings; every case also checks local_error against the oracle."""
    from oracle import dash_oracle as orc
    from paper_2305_18376_b200 import workloads as wl
    from paper_2305_18376_b200.evaluate import local_error
    cfg = wl.scaled(wl.CONFIGS[name], **kw)
    stream_parity(cfg)
    stream = wl.make_stream(cfg)
    ps = wl.planted_state(stream)
    gpu, cpu = gpu_state_from_planted(ps, passes=cfg.passes), oracle_from_planted(ps, passes=cfg.passes)
    batch = next(stream.batches())
    res, ref = gpu.update(batch), cpu.update(batch)
    items = [(s, r) for s, r, _ in batch.items()]
    te, per = local_error(items, res.u_new, gpu)
    te_o, per_o = orc.local_error(items, ref["u_new"], {s: cpu.W[cpu.row_of(s)] for s, _ in items}, cpu.V)
    assert abs(te - te_o) <= TOL * abs(te_o)
    assert max(abs(per[s] - per_o[s]) for s, _ in items) <= TOL * max(per_o.values())
