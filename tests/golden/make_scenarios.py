"""Record the INPUT streams of the reference's own test scenarios, plus the
reference's end state on them, so the GPU engine can be put through the same
assertions on a box where /root/reference does not exist.

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_scenarios.py

Scenarios (the reference test each one comes from):

  structure / rows / dormant / residual / parity / resume / json
      /root/reference/pkg/tests/test_stream_engine.py:14-25 ``planted_stream``
      with the seeds and knobs of TestStructure (:29-108),
      TestNormalEquationResiduals (:132-139), TestKernelParity (:205-228) and
      TestCheckpoints (:231-287)
  ledger_*
      TestLedgerOracle.run_with_ledger (:143-203): lambda in {0.4, 0.7, 1.0},
      passes=3, and the first-update stale-V case
  c1_* / c2_*
      test_acceptance.py:60-92 ``random_stream`` drawn with the generators of
      criteria 1 (:96-126, rng 101) and 2 (:129-164, rng 202); the first
      N_C1 / N_C2 draws only, to keep the fixture small
  planted
      criterion 4 (:211-240): noiseless planted tensor, 3,000 ALS sweeps
  c9
      criterion 9 (:416-475): determinism and resume

For every scenario the file holds the initial tensor, every batch (rows, ids,
first steps, cycle spans), the ``initialize`` arguments, and the reference's
state after the last update (V, W, C, D, F, G) -- the latter lets the GPU
tests compare end states with the reference as TestKernelParity compares the
reference's two kernels.  Nothing here is read by the product.
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from p2stream.stream import initialize  # noqa: E402
from p2stream.synth import SynthParams, synthesize  # noqa: E402
from p2stream.tensor import replay  # noqa: E402

N_C1 = 10
N_C2 = 5


def pack(out, name, initial, batches, rank, iters, seed, lam, passes=1, run=True):
    p = f"{name}/"
    out[p + "args"] = np.array([rank, iters, seed, passes], dtype=np.int64)
    out[p + "lam"] = np.float64(lam)
    out[p + "init_ids"] = np.array([s.slice_id for s in initial.slices])
    out[p + "init_first"] = np.array([s.first_time_step for s in initial.slices], dtype=np.int64)
    out[p + "init_counts"] = np.array([s.row_count for s in initial.slices], dtype=np.int64)
    out[p + "init_X"] = np.concatenate([s.rows for s in initial.slices])
    out[p + "n_batches"] = np.int64(len(batches))
    for t, b in enumerate(batches):
        items = list(b.items())
        q = f"{p}b{t}_"
        out[q + "X"] = np.concatenate([rows for _, rows, _ in items])
        out[q + "ids"] = np.array([sid for sid, _, _ in items])
        out[q + "counts"] = np.array([rows.shape[0] for _, rows, _ in items], dtype=np.int64)
        out[q + "new"] = np.array([new for _, _, new in items], dtype=bool)
        first = {ns.slice_id: ns.first_time_step for ns in b.new_slices}
        out[q + "first"] = np.array([first.get(sid, -1) for sid, _, _ in items], dtype=np.int64)
        out[q + "span"] = np.array(b.cycle_span, dtype=np.int64)
        out[q + "index"] = np.int64(b.update_index)
    if run:
        state, info = initialize(initial, rank, iters=iters, seed=seed, forgetting=lam, passes=passes)
        out[p + "ref_init_V"] = state.V.copy()
        out[p + "ref_init_W"] = state.W.copy()
        for b in batches:
            state.update(b)
        for k in ("V", "W", "C", "D", "F", "G"):
            out[p + "ref_" + k] = getattr(state, k).copy()
        out[p + "ref_ids"] = np.array(state.slice_ids)


def planted_stream(seed=0, stagger=0.0, noise=0.05, slices=6, cols=8, rank=3,
                   duration=90, cycle=10, lam=0.7, iters=8, passes=1):
    tensor = synthesize(SynthParams(num_slices=slices, num_columns=cols, rank=rank, duration=duration,
                                    noise=noise, stagger=stagger), seed=seed)
    initial, batches = replay(tensor, 0.3, cycle)
    return initial, batches, dict(rank=rank, iters=iters, seed=seed, lam=lam, passes=passes)


def random_stream(rng, min_updates=10, stagger_choices=(0.0, 0.4)):
    """Same draw order as test_acceptance.py:60-92 (so the seeded sequence of
    streams is the reference's), without fitting."""
    while True:
        slices = int(rng.integers(3, 31))
        rank = int(rng.integers(1, 6))
        cols = int(rng.integers(max(4, 3 * rank), 21))
        cycle = int(rng.integers(3, 11))
        duration = int(np.ceil(cycle * (min_updates + 2) / 0.7)) + 1
        params = SynthParams(num_slices=slices, num_columns=cols, rank=rank, duration=duration,
                             noise=float(rng.uniform(0.05, 0.2)), stagger=float(rng.choice(stagger_choices)))
        seed = int(rng.integers(0, 2**31))
        try:
            tensor = synthesize(params, seed)
            initial, batches = replay(tensor, 0.3, cycle)
            if min(s.row_count for s in initial.slices) < rank:
                continue
            if len(batches) < min_updates:
                continue
        except ValueError:
            continue
        lam = float(rng.choice([0.5, 0.7, 0.9, 1.0]))
        # the reference fits here (its rng is not touched by the fit)
        return initial, batches, dict(rank=rank, iters=10, seed=seed, lam=lam)


def main():
    out = {}
    for name, kw in {
        "structure": dict(stagger=0.6, seed=3),
        "rows": dict(seed=1),
        "dormant": dict(seed=2),
        "residual": dict(seed=6, stagger=0.5, noise=0.1),
        "parity": dict(seed=14, stagger=0.5, noise=0.1),
        "json": dict(seed=15),
        "resume": dict(seed=18, stagger=0.5),
    }.items():
        initial, batches, a = planted_stream(**kw)
        pack(out, name, initial, batches, **a)

    for tag, seed, lam, passes in (("ledger_l04", 11, 0.4, 1), ("ledger_l07", 11, 0.7, 1),
                                   ("ledger_l10", 11, 1.0, 1), ("ledger_p3", 12, 0.6, 3)):
        tensor = synthesize(SynthParams(num_slices=5, num_columns=6, rank=2, duration=60, noise=0.05,
                                        stagger=0.4), seed=seed)
        initial, batches = replay(tensor, 0.3, 8)
        pack(out, tag, initial, batches, rank=2, iters=6, seed=seed, lam=lam, passes=passes)

    tensor = synthesize(SynthParams(num_slices=4, num_columns=6, rank=2, duration=40, noise=0.05), seed=13)
    initial, batches = replay(tensor, 0.5, 10)
    pack(out, "ledger_stale", initial, batches[:1], rank=2, iters=6, seed=0, lam=1.0)

    rng = np.random.default_rng(101)
    for n in range(N_C1):
        initial, batches, a = random_stream(rng)
        pack(out, f"c1_{n}", initial, batches, **a)
    rng = np.random.default_rng(202)
    for n in range(N_C2):
        initial, batches, a = random_stream(rng)
        pack(out, f"c2_{n}", initial, batches, **a)

    tensor = synthesize(SynthParams(num_slices=20, num_columns=15, rank=3, duration=250, init_window=50), seed=3)
    initial, batches = replay(tensor, 0.2, 20)
    assert len(batches) == 10
    pack(out, "planted", initial, batches, rank=3, iters=3000, seed=0, lam=1.0)

    tensor = synthesize(SynthParams(num_slices=6, num_columns=8, rank=3, duration=200, noise=0.05, stagger=0.4),
                        seed=4)
    initial, batches = replay(tensor, 0.3, 10)
    pack(out, "c9", initial, batches, rank=3, iters=6, seed=4, lam=0.7)

    out["names"] = np.array(sorted({k.split("/")[0] for k in out if "/" in k}))
    path = HERE / "scenarios.npz"
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({path.stat().st_size / 1e6:.2f} MB, {len(out)} arrays)")


if __name__ == "__main__":
    main()
