"""Generate the golden vectors that pin oracle/ to the reference.

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports the reference package ``p2stream`` read-only from
/root/reference/pkg/src, feeds it seeded streams from
``paper_2305_18376_b200.workloads`` (inputs are stored too, so nothing needs
regenerating), and records what the reference returns:

  tiny_stream.npz   BASELINE configs[0] (K0=100, J=20, R=5, lambda=1.0,
                    10 updates): initial tensor, reference ``initialize``
                    (parafac2_als losses / Q_k / factors + init_helpers) and,
                    after every ``StreamState.update``, u_new, W, C, D, F, G,
                    V, v_used and ``local_error``.
  multipass.npz     passes=3, lambda=0.6 on a planted state, numba path and
                    numpy path (USE_FAST_KERNEL False) both recorded.
  edge.npz          new slices shorter than R, single-row slices, batches of
                    only new / only existing slices, R=32 wide-ish state.
  kernel.npz        direct ``group_update`` calls (numba kernel) on random
                    inputs, for the bit-level check of oracle/group_update.c.
  ckpt_ref.json     reference ``save_state`` checkpoints (JSON and npz) of a
  ckpt_ref.npz      planted tiny state after 3 updates, with column stats;
  ckpt.npz          the 2 updates that follow (resume trajectory) and a causal
                    ``normalize_batch`` chain (normalised rows + final stats).
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import p2stream  # noqa: E402
import p2stream.stream as ref_stream  # noqa: E402
from p2stream._kernels import group_update as ref_group_update  # noqa: E402
from p2stream.evaluate import local_error as ref_local_error  # noqa: E402

from paper_2305_18376_b200 import workloads as wl  # noqa: E402


def to_ref_batch(batch):
    return p2stream.UpdateBatch(
        batch.update_index,
        dict(batch.existing_rows),
        [p2stream.NewSlice(ns.slice_id, ns.rows, ns.first_time_step) for ns in batch.new_slices],
        batch.cycle_span,
    )


def pack_batch(batch):
    """Batch as flat arrays: X rows in items() order, ids, row counts, is_new."""
    ids, counts, new, xs = [], [], [], []
    for sid, rows, is_new in batch.items():
        ids.append(sid)
        counts.append(rows.shape[0])
        new.append(is_new)
        xs.append(rows)
    return np.concatenate(xs), np.array(ids), np.array(counts), np.array(new)


def record_updates(state, batches, out, prefix):
    for t, batch in enumerate(batches):
        X, ids, counts, new = pack_batch(batch)
        out[f"{prefix}b{t}_X"] = X
        out[f"{prefix}b{t}_ids"] = ids
        out[f"{prefix}b{t}_counts"] = counts
        out[f"{prefix}b{t}_new"] = new
        res = state.update(to_ref_batch(batch))
        out[f"{prefix}u{t}_U"] = np.concatenate([res.u_new[sid] for sid in ids])
        for name in ("W", "C", "D", "F", "G", "V"):
            out[f"{prefix}u{t}_{name}"] = getattr(state, name).copy()
        out[f"{prefix}u{t}_v_used"] = res.v_used.copy()
        items = [(sid, rows) for sid, rows, _ in batch.items()]
        te, per = ref_local_error(items, res.u_new, state)
        out[f"{prefix}u{t}_local_error"] = np.array(te)
        out[f"{prefix}u{t}_slice_error"] = np.array([per[sid] for sid in ids])
        out[f"{prefix}u{t}_slice_ids"] = np.array(state.slice_ids)
    out[f"{prefix}n_updates"] = np.array(len(batches))


def planted_ref_state(stream):
    ps = wl.planted_state(stream)
    return p2stream.StreamState(
        slice_ids=list(ps["slice_ids"]),
        u_blocks={sid: [np.zeros((0, stream.cfg.R))] for sid in ps["slice_ids"]},
        W=ps["W"].copy(), V=ps["V"].copy(), C=ps["C"].copy(), D=ps["D"].copy(),
        F=ps["F"].copy(), G=ps["G"].copy(), forgetting=ps["forgetting"],
        passes=stream.cfg.passes,
    ), ps


def save_planted(out, prefix, ps):
    for k in ("W", "V", "C", "D", "F", "G"):
        out[f"{prefix}init_{k}"] = ps[k]
    out[f"{prefix}init_ids"] = np.array(ps["slice_ids"])
    out[f"{prefix}forgetting"] = np.array(ps["forgetting"])


def make_tiny():
    stream = wl.make_stream("tiny")
    cfg = stream.cfg
    init = stream.initial_tensor()
    out = {}
    out["init_X"] = np.concatenate([s.rows for s in init.slices])
    out["init_counts"] = np.array([s.row_count for s in init.slices])
    out["init_ids"] = np.array(init.slice_ids)
    ref_init = p2stream.IrregularTensor(
        p2stream.SliceMatrix(s.slice_id, s.rows) for s in init.slices)
    state, info = p2stream.initialize(ref_init, cfg.R, iters=10, seed=cfg.seed,
                                      forgetting=cfg.forgetting)
    out["als_losses"] = np.array(info.losses)
    out["als_Q"] = np.concatenate([info.projections[sid] for sid in init.slice_ids])
    fs = state.factor_set()
    out["als_U"] = np.concatenate([fs.U[sid] for sid in init.slice_ids])
    out["als_W"] = fs.W
    out["als_V"] = fs.V
    for name in ("C", "D", "F", "G"):
        out[f"init_{name}"] = getattr(state, name).copy()
    out["R"] = np.array(cfg.R)
    out["forgetting"] = np.array(cfg.forgetting)
    # ALS with tol=0 (fixed sweep count, the refit-baseline mode evaluate.py:219-221)
    f0 = p2stream.parafac2_als(ref_init, cfg.R, iters=4, seed=7, tol=0.0, return_info=True)
    out["als_tol0_losses"] = np.array(f0[1].losses)
    out["als_tol0_V"] = f0[0].V
    out["als_tol0_W"] = f0[0].W
    record_updates(state, list(stream.batches()), out, "")
    np.savez_compressed(HERE / "tiny_stream.npz", **out)


def make_multipass():
    cfg = wl.scaled(wl.CONFIGS["medium"], K0=12, steps=4, new_slices=2, J=10, R=3,
                    forgetting=0.6, passes=3, seed=21,
                    init_rows=("uniform", 5, 20), add_rows=("uniform", 1, 4),
                    new_rows=("uniform", 2, 9))
    out = {}
    for tag, fast in (("fast_", True), ("numpy_", False)):
        ref_stream.USE_FAST_KERNEL = fast
        try:
            stream = wl.make_stream(cfg)
            state, ps = planted_ref_state(stream)
            save_planted(out, tag, ps)
            out[f"{tag}passes"] = np.array(3)
            record_updates(state, list(stream.batches()), out, tag)
        finally:
            ref_stream.USE_FAST_KERNEL = True
    np.savez_compressed(HERE / "multipass.npz", **out)


def make_edge():
    out = {}
    # (a) daily-like: new slices with fewer rows than R, single-row appends
    cfg = wl.scaled(wl.CONFIGS["daily"], K0=15, steps=5, J=14, R=6, seed=31,
                    init_rows=("loguniform", 6, 60), new_slices=("uniform", 1, 3),
                    new_rows=("uniform", 1, 4))
    stream = wl.make_stream(cfg)
    state, ps = planted_ref_state(stream)
    save_planted(out, "a_", ps)
    record_updates(state, list(stream.batches()), out, "a_")
    # (b) wide-ish rank: R=32, J=48, mixed heights incl. a 70-row new slice
    cfg = wl.scaled(wl.CONFIGS["wide32"], K0=10, steps=3, J=48, R=32, seed=32,
                    new_slices=1, init_rows=("uniform", 40, 80), new_rows=("uniform", 60, 80))
    stream = wl.make_stream(cfg)
    state, ps = planted_ref_state(stream)
    save_planted(out, "b_", ps)
    record_updates(state, list(stream.batches()), out, "b_")
    # (c) only-new and only-existing batches, odd J
    cfg = wl.scaled(wl.CONFIGS["tiny"], K0=6, steps=1, J=7, R=2, seed=33,
                    init_rows=("uniform", 4, 8), forgetting=0.8)
    stream = wl.make_stream(cfg)
    state, ps = planted_ref_state(stream)
    save_planted(out, "c_", ps)
    rng = np.random.default_rng(33)
    only_new = wl.UpdateBatch(1, {}, [wl.NewSlice("n0", rng.standard_normal((3, 7)), 1),
                                      wl.NewSlice("n1", rng.standard_normal((1, 7)), 1)], (1, 1))
    only_old = wl.UpdateBatch(2, {"s000001": rng.standard_normal((2, 7)),
                                  "n1": rng.standard_normal((5, 7))}, [], (2, 2))
    record_updates(state, [only_new, only_old], out, "c_")
    np.savez_compressed(HERE / "edge.npz", **out)


def make_kernel():
    rng = np.random.default_rng(41)
    out = {}
    cases = [(7, 3, 5), (4, 1, 2), (3, 12, 16), (2, 5, 32), (1, 40, 10)]
    for n, (G, I, R) in enumerate(cases):
        xv = rng.standard_normal((G, I, R))
        v = rng.standard_normal((R + 3, R))
        vtv = v.T @ v
        s = rng.uniform(0.2, 1.5, size=(G, R))
        c_old = rng.standard_normal((G, R))
        b = rng.standard_normal((G, R, R + 2))
        d_old = b @ b.transpose(0, 2, 1)
        lam = 0.85
        res = ref_group_update(xv, vtv, s, c_old, d_old, lam, 1e-10)
        for key, val in zip(("xv", "vtv", "s", "c_old", "d_old"), (xv, vtv, s, c_old, d_old)):
            out[f"k{n}_{key}"] = val
        out[f"k{n}_lam"] = np.array(lam)
        for key, val in zip(("u", "us", "c_new", "d_new", "w", "g_fresh", "ok"), res):
            out[f"k{n}_out_{key}"] = np.asarray(val)
    out["n_cases"] = np.array(len(cases))
    np.savez_compressed(HERE / "kernel.npz", **out)


def make_checkpoint():
    from p2stream.tensor import global_stats, normalize_batch
    stream = wl.make_stream("tiny")
    state, ps = planted_ref_state(stream)
    batches = list(stream.batches())
    out = {}
    save_planted(out, "", ps)
    # causal normalisation chain, seeded by the initial tensor's global stats
    init = stream.initial_tensor()
    stats = global_stats(p2stream.IrregularTensor(
        p2stream.SliceMatrix(s.slice_id, s.rows) for s in init.slices))
    for t, batch in enumerate(batches[:4]):
        X, ids, counts, new = pack_batch(batch)
        out[f"nb{t}_X"], out[f"nb{t}_ids"], out[f"nb{t}_counts"], out[f"nb{t}_new"] = X, ids, counts, new
        nb, stats = normalize_batch(to_ref_batch(batch), stats)
        out[f"nb{t}_Xn"] = np.concatenate(
            [nb.existing_rows[sid] for sid in nb.existing_rows] + [ns.rows for ns in nb.new_slices])
    sids = sorted(stats.minimum)
    out["nstats_ids"] = np.array(sids)
    out["nstats_min"] = np.stack([stats.minimum[s] for s in sids])
    out["nstats_max"] = np.stack([stats.maximum[s] for s in sids])
    out["n_norm"] = np.array(4)
    # checkpoint after 3 updates (with the stats), then the resume trajectory
    for batch in batches[:3]:
        state.update(to_ref_batch(batch))
    ref_stream.save_state(state, HERE / "ckpt_ref.json", column_stats=stats)
    ref_stream.save_state(state, HERE / "ckpt_ref.npz", column_stats=stats)
    record_updates(state, batches[3:5], out, "r")
    np.savez_compressed(HERE / "ckpt.npz", **out)


if __name__ == "__main__":
    make_checkpoint()
    make_kernel()
    make_edge()
    make_multipass()
    make_tiny()
    for p in sorted(HERE.glob("*.npz")):
        print(p.name, p.stat().st_size)
