"""Driver for ncu captures: a few device-resident updates of a config at full
size (no timing).  python tools/prof_update.py [config] [updates] [K0]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2305_18376_b200 import workloads as wl  # noqa: E402
from paper_2305_18376_b200.stream import StreamState  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "large"
updates = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = wl.CONFIGS[name]
if len(sys.argv) > 3:
    cfg = wl.scaled(cfg, K0=int(sys.argv[3]))
cfg = wl.scaled(cfg, steps=updates)
dev = torch.device("cuda", 0)
stream = wl.make_stream(cfg, exact=False)
ps = wl.planted_state(stream)
st = StreamState.from_arrays(ps, device=dev)
R, J = cfg.R, cfg.J
H, V = wl.true_factors(cfg)
gen = torch.Generator(device=dev)
gen.manual_seed(7)
sch = stream.schedule
K = cfg.K0
for t in range(updates):
    add, new = sch.adds[t], sch.new_len[t]
    counts = np.concatenate([add, new]).astype(np.int64)
    N = int(counts.sum())
    X = 0.1 * torch.randn((N, J), generator=gen, device=dev, dtype=torch.float64)
    st.update_packed(X, counts, np.arange(K, dtype=np.int32), [wl.slice_id(K + i) for i in range(len(new))])
    K += len(new)
torch.cuda.synchronize()
st.check()
print("done", name, updates)
