"""Workload for compute-sanitizer (memcheck / racecheck / synccheck): every
kernel family of the update path on small streams, PDL on (the default).

    compute-sanitizer --tool racecheck python tools/sanitize_run.py

Runs: the tiny golden config; a reduced large stream (big + small slices on
the fused path, R=16, FP64 and the FP32 data mode, 2 passes); reduced wide
streams (R=10 J=1024, R=32, R=64); daily-shaped (1-row appends); local_error,
init_helpers and one ALS fit.  Checks nothing numerically (the pytest suite
does); the sanitizer's report is the output."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2305_18376_b200 import workloads as wl  # noqa: E402
from paper_2305_18376_b200.evaluate import local_error  # noqa: E402
from paper_2305_18376_b200.stream import StreamState, initialize  # noqa: E402


def drive(cfg, dtype=torch.float64, err=True):
    stream = wl.make_stream(cfg, exact=False)
    st = StreamState.from_arrays(wl.planted_state(stream), dtype=dtype)
    for b in stream.batches():
        res = st.update(b)
        if err:
            local_error([(s, r) for s, r, _ in b.items()], res.u_new, st)
    torch.cuda.synchronize()
    print(f"ok {cfg.name} K0={cfg.K0} R={cfg.R} J={cfg.J} passes={cfg.passes} {dtype}", flush=True)


def main():
    which = sys.argv[1:] or ["tiny", "large", "large32", "large2", "daily", "wide10", "wide32", "wide64", "als"]
    if "tiny" in which:
        drive(wl.scaled(wl.CONFIGS["tiny"], steps=3))
    if "large" in which:
        drive(wl.scaled(wl.CONFIGS["large"], K0=600, steps=2, new_slices=3, add_rows=("uniform", 1, 100)))
    if "large32" in which:
        drive(wl.scaled(wl.CONFIGS["large"], K0=600, steps=2, new_slices=3), dtype=torch.float32)
    if "large2" in which:
        drive(wl.scaled(wl.CONFIGS["large"], K0=300, steps=2, new_slices=2, passes=2))
    if "daily" in which:
        drive(wl.scaled(wl.CONFIGS["daily"], K0=400, steps=3))
    for name in ("wide10", "wide32", "wide64"):
        if name in which:
            drive(wl.scaled(wl.CONFIGS[name], K0=60, steps=2, new_slices=2), err=(name == "wide10"))
    if "als" in which:
        cfg = wl.scaled(wl.CONFIGS["medium"], K0=40, steps=1)
        stream = wl.make_stream(cfg)
        initialize(stream.initial_tensor(), cfg.R, iters=2, seed=0)
        torch.cuda.synchronize()
        print("ok als", flush=True)
    print("sanitize_run done")


if __name__ == "__main__":
    main()
