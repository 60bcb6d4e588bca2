"""Debug: per-update errors of the GPU update vs the oracle, split by small /
big slices (rows <= 32 / > 32).  python tools/dbg_smallx.py [config] [K0] [steps]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402

from golden_io import rel  # noqa: E402
from oracle import dash_oracle as orc  # noqa: E402
from paper_2305_18376_b200 import _native as nat  # noqa: E402
from paper_2305_18376_b200 import workloads as wl  # noqa: E402
from paper_2305_18376_b200.stream import StreamState  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "medium"
K0 = int(sys.argv[2]) if len(sys.argv) > 2 else 150
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
kw = dict(K0=K0, steps=steps)
if name == "large":
    kw["new_slices"] = 3
cfg = wl.scaled(wl.CONFIGS[name], **kw)
orc.build_c()
stream = wl.make_stream(cfg, exact=False)
ps = wl.planted_state(stream)
R = cfg.R
gpu = StreamState.from_arrays(ps)
cpu = orc.OracleStreamState(ps["slice_ids"], {s: [] for s in ps["slice_ids"]}, ps["W"], ps["V"], ps["C"],
                            ps["D"], ps["F"], ps["G"], ps["forgetting"])
for t, b in enumerate(stream.batches()):
    res = gpu.update(b)
    ref = cpu.update(b)
    flags = nat.lib().dash_ctx_path_flags(gpu._ctx)
    ids = [s for s, _, _ in b.items()]
    n = {s: r.shape[0] for s, r, _ in b.items()}
    small = [s for s in ids if n[s] <= 32]
    big = [s for s in ids if n[s] > 32]
    out = {"flags": flags, "M": len(ids), "small": len(small), "big": len(big)}
    for tag, grp in (("s", small), ("b", big)):
        if not grp:
            continue
        out["U" + tag] = rel(np.concatenate([res.u_new[s] for s in grp]), np.concatenate([ref["u_new"][s] for s in grp]))
        rows = [gpu.row_of(s) for s in grp]
        out["W" + tag] = rel(gpu.W[rows], cpu.W[rows])
        out["C" + tag] = rel(gpu.C[rows], cpu.C[rows])
        out["D" + tag] = rel(gpu.D[rows], cpu.D[rows])
        if tag == "s":
            worst = max(grp, key=lambda s: np.abs(res.u_new[s] - ref["u_new"][s]).max())
            out["worst_small"] = (worst, n[worst], ids.index(worst))
    for nm in ("F", "G", "V"):
        out[nm] = rel(getattr(gpu, nm), getattr(cpu, nm))
    print(t, {k: (f"{v:.2e}" if isinstance(v, float) else v) for k, v in out.items()}, flush=True)
