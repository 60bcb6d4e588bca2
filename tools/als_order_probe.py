"""Does the daily ALS sweep time depend on what ran before it in the process?"""
import sys
sys.path.insert(0, '.')
import torch
import bench
dev = torch.device("cuda", 0)
order = sys.argv[1:] or ["medium", "daily", "daily"]
for name in order:
    r = bench.als_timing(name, dev, iters=3)
    print(name, round(r["sweep_ms"], 2), "ms/sweep; fit(1 sweep)", round(r["fit_ms_1_sweep"], 1), flush=True)
