"""Timed loop like bench.py's (large config, device-resident batches): GPU
events around the loop vs the host time of every update_packed call.
python tools/host_vs_gpu.py [steps] [K0]"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2305_18376_b200 import workloads as wl  # noqa: E402
from paper_2305_18376_b200.stream import StreamState  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 12
cfg = wl.CONFIGS["large"]
if len(sys.argv) > 2:
    cfg = wl.scaled(cfg, K0=int(sys.argv[2]))
cfg = wl.scaled(cfg, steps=steps)
dev = torch.device("cuda", 0)
stream = wl.make_stream(cfg, exact=False)
st = StreamState.from_arrays(wl.planted_state(stream), device=dev)
gen = torch.Generator(device=dev)
gen.manual_seed(7)
sch = stream.schedule
K = cfg.K0
batches = []
for t in range(steps):
    add, new = sch.adds[t], sch.new_len[t]
    counts = np.concatenate([add, new]).astype(np.int64)
    X = 0.1 * torch.randn((int(counts.sum()), cfg.J), generator=gen, device=dev, dtype=torch.float64)
    batches.append((X, counts, np.arange(K, dtype=np.int32), [wl.slice_id(K + i) for i in range(len(new))]))
    K += len(new)
st.reserve_u_history(sum(b[0].shape[0] for b in batches))
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
host = []
e[0].record()
for t, b in enumerate(batches):
    h0 = time.perf_counter()
    st.update_packed(*b)
    host.append(1e3 * (time.perf_counter() - h0))
    e[t + 1].record()
torch.cuda.synchronize()
gpu = [e[t].elapsed_time(e[t + 1]) for t in range(steps)]
st.check()
print("host ms:", " ".join(f"{x:.2f}" for x in host))
print("gpu  ms:", " ".join(f"{x:.2f}" for x in gpu))
