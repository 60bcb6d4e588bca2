"""Wall time of the drop-in StreamState.update(UpdateBatch) at a config (host
batches of per-slice numpy arrays, as a reference user calls it), with a
profile of where the host time goes.  python tools/dropin_probe.py [config] [steps]"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2305_18376_b200 import workloads as wl  # noqa: E402
from paper_2305_18376_b200.stream import StreamState  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "large"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = wl.CONFIGS[name]
arrays, gen = bench.host_stream(cfg, steps)
t0 = time.perf_counter()
batches = [b for b, _ in gen()]
print(f"host batch generation {time.perf_counter() - t0:.1f} s")
st = StreamState.from_arrays(arrays, device="cuda")
st.update(batches[0])
torch.cuda.synchronize()
prof = cProfile.Profile()
for b in batches[1:]:
    t0 = time.perf_counter()
    prof.enable()
    st.update(b)
    prof.disable()
    torch.cuda.synchronize()
    print(f"update() wall {1e3 * (time.perf_counter() - t0):.1f} ms")
pstats.Stats(prof).sort_stats("cumulative").print_stats(18)
