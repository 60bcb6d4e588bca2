"""One parafac2_als fit at a BASELINE shape on a device tensor (for ncu launch
lists).  python tools/als_probe.py [medium|daily] [iters]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "medium"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
print(bench.als_timing(name, torch.device("cuda", 0), iters=iters))
