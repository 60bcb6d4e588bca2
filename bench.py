#!/usr/bin/env python
"""Benchmark of the DASH per-update step on B200 (BASELINE.json metric:
"update-step latency and X elements/s at 1/2/4/8 B200; % of HBM roofline").

Workload: the "large" stream of BASELINE.json configs[3] -- K0 = 50,000 slices,
J = 128, R = 16, FP64, lambda = 0.95; every update appends U[1,8] rows to every
active slice and registers 500 new slices of U[200,2000] rows (~0.79 M rows,
~0.81 GB of X per update).  Synthetic data from the planted generator
(workloads.py), drawn on the device; initial state planted in closed form.

A "step" = one StreamState update (all kernels of the pass loop) over one
batch already resident in HBM.  value = X elements (N*J) processed per second
over the timed steps (whole job; max-over-ranks device time).  ms_per_step is
the update-step latency.  Each step's batch is 0.81 GB > 126 MB L2, so the
timed loop never re-reads a cached input ("inputs larger than L2").

e2e: the same metric through the public API with host buffers: pinned host X
-> H2D -> update -> D2H of U_new and v_used, all inside the timed region.

--impl reference: the reference algorithm on the host CPU (oracle/ port of
p2stream's update: numpy/OpenBLAS + the C restatement of the numba kernel),
same workload and metric, rank 0 only.

Multi-GPU (torchrun): slices are partitioned over ranks (slice k -> rank
k % world); each rank runs the per-slice phase on its shard and the F/G fresh
sums are all-reduced with NCCL once per pass before the replicated V solve
(strong scaling: the total stream is fixed).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIG_NAME = "large"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="dash", choices=["dash", "reference"])
    ap.add_argument("--config", default=CONFIG_NAME)
    ap.add_argument("--K0", type=int, default=None, help="override K0 (smoke runs)")
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--no-fp32", dest="fp32", action="store_false",
                    help="skip the FP32 data-mode measurement")
    ap.add_argument("--dropin-steps", type=int, default=3,
                    help="timed StreamState.update(UpdateBatch) calls on host batches (0: skip)")
    ap.add_argument("--parity-steps", type=int, default=2,
                    help="full-size updates of this config checked against the CPU oracle (0: skip)")
    ap.add_argument("--no-als", dest="als", action="store_false",
                    help="skip the parafac2_als sweep timing (medium, daily)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# stream schedule shared by both arms (host RNG; identical for every rank)
# ---------------------------------------------------------------------------
class Schedule:
    def __init__(self, cfg, steps, seed):
        self.cfg = cfg
        rng = np.random.default_rng([seed, 11])
        from paper_2305_18376_b200.workloads import _draw
        self.adds, self.new_len = [], []
        active = cfg.K0
        for _ in range(steps):
            self.adds.append(_draw(rng, cfg.add_rows, active).astype(np.int64))
            L = int(_draw(rng, cfg.new_slices, 1)[0])
            self.new_len.append(_draw(rng, cfg.new_rows, L).astype(np.int64))
            active += L


def ownership(cfg, sched, world):
    """Owner rank of every slice that will ever exist, by the engine's own
    placement rule (distributed.Placement: initial slices by position, each
    new slice to the rank with the least rows in the update that brings it).
    Computed identically on every rank from the shared schedule."""
    from paper_2305_18376_b200.distributed import owner_of_index, place_counts
    n_all = cfg.K0 + sum(len(n) for n in sched.new_len)
    owner = np.full(n_all, -1, dtype=np.int64)
    owner[:cfg.K0] = [owner_of_index(k, world) for k in range(cfg.K0)]
    n_owned = [int(v) for v in np.bincount(owner[:cfg.K0], minlength=world)]
    active = cfg.K0
    for add, new_len in zip(sched.adds, sched.new_len):
        load = np.bincount(owner[:active], weights=add, minlength=world)
        owner[active:active + len(new_len)] = place_counts(world, n_owned, load, new_len)
        active += len(new_len)
    return owner


def algorithmic_bytes(N, J, R, M_old, L, b=8):
    """bytes of one update (read X once, write U, per-slice
    state r/w, new-slice state, F/V/G)."""
    return b * (N * J + N * R + 2 * M_old * (R * R + 2 * R) + L * (R * R + 2 * R)
                + 3 * J * R + 2 * R * R)


def algorithmic_flops(N, J, R, M):
    return 4 * N * J * R + N * (3 * R * R + 2 * R) + M * (4 * R ** 3 / 3 + 4 * R * R)


SMALL_ROWS = 32  # csrc/dash_update.cu kSmallRows: slices with more rows go to k_bigx / k_big


def batch_stats(batches):
    """Average rows / existing / new slices per update, split small vs big."""
    acc = dict(N=0.0, Ns=0.0, Mos=0.0, Ls=0.0, Nb=0.0, Mob=0.0, Lb=0.0)
    for b in batches:
        c = np.asarray(b["counts"])
        new = np.arange(len(c)) >= b["M_old"]
        small = c <= SMALL_ROWS
        acc["N"] += c.sum()
        for k, m in (("s", small), ("b", ~small)):
            acc["N" + k] += c[m].sum()
            acc["Mo" + k] += (m & ~new).sum()
            acc["L" + k] += (m & new).sum()
    return {k: v / max(len(batches), 1) for k, v in acc.items()}


def kernel_bytes(phase, st, J, R, nsplit, b=8, bigx=False):
    """Algorithmic bytes per launch of each kernel (DESIGN.md table).  With the
    fused big-slice path (bigx) the XV / F GEMMs stream only the small slices'
    rows and "big" reads the big slices' rows once (X in, U out, state)."""
    N = st["Ns"] if bigx else st["N"]
    if phase == "xv":        # read X, V; write XV
        return b * (N * J + N * R + J * R)
    if phase == "fgemm":     # read X, US; write one J x R slot per CTA
        return b * (N * J + N * R + nsplit * J * R)
    if phase == "big" and bigx:  # read X once; write U; per-slice W/C/D r/w (new: write only)
        return b * (st["Nb"] * J + st["Nb"] * R + st["Mob"] * (2 * R * R + 4 * R) + st["Lb"] * (R * R + 2 * R))
    if phase in ("slices", "big"):  # read XV; write U, US; per-slice W/C/D r/w (new: write only)
        k = "s" if phase == "slices" else "b"
        return b * (3 * st["N" + k] * R + st["Mo" + k] * (2 * R * R + 4 * R) + st["L" + k] * (R * R + 2 * R))
    return 0


def kernel_flops(phase, st, J, R, bigx=False):
    """FP64 flops per launch of the DMMA kernels: the fused big-slice kernel (XV = X V,
    P = X^T U: 2 N J R each; U = XV Ms^T and U^T U: 2 N R^2 each) and the two
    streaming contractions."""
    if phase == "big" and bigx:
        return 4 * st["Nb"] * J * R + 4 * st["Nb"] * R * R
    if phase in ("xv", "fgemm"):  # one streaming contraction each (DMMA): binds at large R (wide32 / wide64)
        return 2 * (st["Ns"] if bigx else st["N"]) * J * R
    return 0


FP64_TENSOR_PEAK = 37.1  # TFLOP/s, DMMA, measured on this pool's B200 (profiles/r01_fp64_peak.md)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_traffic(phase, config=CONFIG_NAME):
    """dram bytes per launch from a committed `ncu --set full` capture of this
    config (profiles/ncu_traffic.json: {config: {phase: bytes}}); None if that
    config / kernel was not captured."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    return d.get(config, {}).get(phase)


def workload_config(cfg, sched, t0, t1, parallelism):
    """The workload as both arms report it (same keys, same numbers: the row
    counts come from the shared seeded Schedule over the timed steps)."""
    def law(x):
        return list(x)
    n = [int(sched.adds[t].sum() + sched.new_len[t].sum()) for t in range(t0, t1)]
    m = [int(len(sched.adds[t]) + len(sched.new_len[t])) for t in range(t0, t1)]
    return {"workload": cfg.name, "K0": cfg.K0, "J": cfg.J, "R": cfg.R, "lambda": cfg.forgetting,
            "passes": cfg.passes, "init_rows": law(cfg.init_rows), "add_rows_per_slice": law(cfg.add_rows),
            "new_slices": law(cfg.new_slices), "new_slice_rows": law(cfg.new_rows),
            "rows_per_update": sum(n) / max(len(n), 1), "slices_per_update": sum(m) / max(len(m), 1),
            "l2": "inputs larger than L2" if sum(n) / max(len(n), 1) * cfg.J * 8 > 126e6
                  else "batches smaller than L2: device-resident X of every step is distinct",
            "parallelism": parallelism}


def roofline_of(dom, per_kernel, achieved, peak, peak_kind, per_launch_ms, kb, config=CONFIG_NAME):
    """Roofline of the dominant kernel: its binding roof (HBM bytes, or FP64
    tensor flops for the DMMA-bound fused big-slice kernel, whichever fraction
    is higher), with the other roof alongside."""
    pk = per_kernel.get(dom, {})
    hbm = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
           "frac": achieved / peak, "traffic": ncu_traffic(dom, config), "peak_source": peak_kind,
           "per_launch_ms": per_launch_ms, "alg_bytes_per_launch": kb}
    if pk.get("tflops") and pk["frac_fp64_tensor"] > hbm["frac"]:
        return {"bound": "tensor", "kernel": dom, "achieved": pk["tflops"], "peak": FP64_TENSOR_PEAK,
                "unit": "TFLOP/s", "frac": pk["frac_fp64_tensor"], "traffic": ncu_traffic(dom, config),
                "peak_source": "measured FP64 DMMA peak (profiles/r01_fp64_peak.md)",
                "per_launch_ms": per_launch_ms, "alg_flops_per_launch": pk["alg_flops"],
                "hbm": {"achieved": achieved, "peak": peak, "frac": achieved / peak, "alg_bytes_per_launch": kb}}
    return hbm


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2305_18376_b200 import _native as nat
    from paper_2305_18376_b200 import workloads as wl
    from paper_2305_18376_b200.distributed import ShardedStream
    from paper_2305_18376_b200.stream import StreamState

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # Validation knobs for the multi-rank code path on a single-GPU box (not
    # for measurement): DASH_BENCH_DEVICE pins every rank to one device,
    # DASH_BENCH_BACKEND=gloo exchanges the F/G sums on the host.
    if "DASH_BENCH_DEVICE" in os.environ:
        local = int(os.environ["DASH_BENCH_DEVICE"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("DASH_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    cfg = wl.CONFIGS[args.config]
    if args.K0:
        cfg = wl.scaled(cfg, K0=args.K0)
    J, R = cfg.J, cfg.R
    prof_steps = 3  # separate profiled steps for the per-phase breakdown (events kept out of the timed loop)
    total_steps = args.warmup + args.steps + prof_steps + args.e2e_steps
    sched = Schedule(cfg, total_steps, cfg.seed)
    H, V = wl.true_factors(cfg)
    # true per-slice weights for every slice that will ever exist
    n_all = cfg.K0 + sum(len(n) for n in sched.new_len)
    w_true = np.random.default_rng([cfg.seed, 12]).uniform(size=(n_all, R))
    # planted initial state (closed form, see workloads.planted_state) for owned slices
    owner = ownership(cfg, sched, world)
    own0 = np.nonzero(owner[:cfg.K0] == rank)[0].astype(np.int64)
    D0 = H.T @ H
    vtv = V.T @ V
    Wl = w_true[own0]
    G_all = np.einsum("kr,rz,kz->rz", w_true[:cfg.K0], D0, w_true[:cfg.K0])
    G_all = (G_all + G_all.T) / 2.0
    arrays = {
        "slice_ids": [wl.slice_id(int(k)) for k in own0],
        "W": Wl, "V": V, "C": np.einsum("rz,kz,zr->kr", D0, Wl, vtv),
        "D": np.broadcast_to(D0, (len(own0), R, R)).copy(),
        "F": V @ G_all, "G": G_all, "forgetting": cfg.forgetting, "passes": cfg.passes,
    }
    state = StreamState.from_arrays(arrays, device=dev)
    engine = ShardedStream(state, rank=rank, world=world) if world > 1 else None

    Hd = torch.as_tensor(H, device=dev)
    Vd = torch.as_tensor(V, device=dev)
    wd = torch.as_tensor(w_true, device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(cfg.seed * 1000 + 17)

    # per-step local batches, generated on the device before timing
    active = list(range(cfg.K0))
    local_row = {int(k): i for i, k in enumerate(own0)}  # global slice -> local state row
    batches = []
    for t in range(total_steps):
        add = sched.adds[t]
        ex = [k for k in active if owner[k] == rank]
        ex_counts = add[np.array(ex, dtype=np.int64)] if ex else np.zeros(0, np.int64)
        base = len(active)
        new = [base + i for i in range(len(sched.new_len[t])) if owner[base + i] == rank]
        new_counts = sched.new_len[t][np.array(new, dtype=np.int64) - base] if new else np.zeros(0, np.int64)
        active.extend(range(base, base + len(sched.new_len[t])))
        ex_rows = np.array([local_row[k] for k in ex], dtype=np.int32)
        for k in new:
            local_row[k] = len(local_row)
        counts = np.concatenate([ex_counts, new_counts]).astype(np.int64)
        slices_of_rows = torch.as_tensor(np.repeat(np.array(ex + new, dtype=np.int64), counts), device=dev)
        N = int(counts.sum())
        q = torch.randn((N, R), generator=gen, device=dev, dtype=torch.float64) / np.sqrt(1100.0)
        X = ((q @ Hd) * wd[slices_of_rows]) @ Vd.T
        X += 0.1 * torch.randn((N, J), generator=gen, device=dev, dtype=torch.float64)
        del q, slices_of_rows
        batches.append({"X": X, "counts": counts, "ex_rows": ex_rows, "new": [wl.slice_id(k) for k in new],
                        "N": N, "M_old": len(ex), "L": len(new)})

    def step(b):
        if engine is not None:
            return engine.update_packed(b["X"], b["counts"], b["ex_rows"], b["new"])
        return state.update_packed(b["X"], b["counts"], b["ex_rows"], b["new"])

    def barrier():
        if world > 1:
            dist.barrier()

    # the U history (kept, as the reference keeps u_blocks) gets its device
    # room up front, so no update in the timed loop allocates
    state.reserve_u_history(sum(b["N"] for b in batches))
    # warm-up
    for t in range(args.warmup):
        step(batches[t])
    torch.cuda.synchronize()
    state.check()

    # timed region (device-resident batches)
    L = nat.lib()
    timed = batches[args.warmup:args.warmup + args.steps]
    sampler = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.3)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    e0.record(stream)
    for b in timed:
        step(b)
        launches += state.last_launches
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    fallbacks = L.dash_ctx_fallbacks(state._ctx, nat.stream_ptr(), 1)
    # per-phase breakdown: separate steps with CUDA events around every launch
    import ctypes
    profiled = batches[args.warmup + args.steps:args.warmup + args.steps + prof_steps]
    torch.cuda.synchronize()
    L.dash_ctx_set_profiling(state._ctx, 1)
    for b in profiled:
        step(b)
    torch.cuda.synchronize()
    nph = len(nat.PHASES)
    ms_arr = (ctypes.c_double * nph)()
    cnt_arr = (ctypes.c_int32 * nph)()
    L.dash_ctx_phase_ms(state._ctx, ms_arr, cnt_arr, nph)
    L.dash_ctx_set_profiling(state._ctx, 0)
    state.check()
    # the per-update fitness (evaluate.local_error) on the device-resident batch the
    # last profiled update just consumed: the reference's comment asks that it stay cheap next to
    # the update it measures -- timed here (second pass over X: row errors on DMMA tiles + sums)
    fitness = None
    if profiled:
        from paper_2305_18376_b200.evaluate import local_error_device
        lb = profiled[-1]
        _, _, meta, Xl, Nl, Ul = state._last
        rp_h = meta.host_row_ptr().copy()
        sr_d = meta[1]
        local_error_device(Xl, Nl, rp_h, sr_d, Ul, state, row_ptr_dev=meta[0])  # warm-up
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        f0.record(stream)
        for _ in range(reps):
            local_error_device(Xl, Nl, rp_h, sr_d, Ul, state, row_ptr_dev=meta[0])
        f1.record(stream)
        torch.cuda.synchronize()
        fit_ms = f0.elapsed_time(f1) / reps
        fb = 8 * (lb["N"] * J + lb["N"] * R + J * R)
        fitness = {"ms_per_update": fit_ms, "alg_bytes": fb, "gbs": fb / (fit_ms / 1e3) / 1e9,
                   "what": "local_error of one update's batch (device-resident X, U_new; per-slice MAD + tensor mean)"}
    t_ms = e0.elapsed_time(e1)
    t_max = t_ms
    if world > 1:
        tt = torch.tensor([t_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    elems_local = sum(b["N"] for b in timed) * J
    elems = elems_local
    if world > 1:
        te = torch.tensor([elems_local], device=dev, dtype=torch.float64)
        dist.all_reduce(te)
        elems = float(te.item())
    value = elems / (t_max / 1e3)
    ms_per_step = t_max / len(timed)

    # FP32 data mode (north_star: optional, reported separately): a second
    # state fed the same batches rounded to FP32; device-resident timing of the
    # same K steps, then the same e2e protocol with FP32 host buffers.
    fp32 = None
    if args.fp32:
        fp32 = run_fp32_arm(args, arrays, batches, dev, stream, world, J, R, prof_steps, barrier)

    # e2e through the public API with host buffers: HostPipeline uploads batch
    # t+1 (pinned host -> HBM) and reads back batch t-1's U / v_used while
    # batch t is updated; every step's H2D and D2H lie inside the timed region.
    from paper_2305_18376_b200.stream import HostPipeline
    e2e_b = batches[args.warmup + args.steps + prof_steps:]
    pins = []
    for b in e2e_b:
        hp = torch.empty_like(b["X"], device="cpu").pin_memory()
        hp.copy_(b["X"])
        pins.append(hp)
        b["X"] = None  # device copy no longer needed
    maxN = max((b["N"] for b in e2e_b), default=1)
    Uh = [torch.empty((maxN, R), dtype=torch.float64).pin_memory() for _ in range(2)]
    vh = [torch.empty((J, R), dtype=torch.float64).pin_memory() for _ in range(2)]
    pipe = HostPipeline(engine if engine is not None else state, maxN, J, device=dev)
    torch.cuda.synchronize()
    barrier()
    h2d = d2h = 0
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    pipe.start()
    staged = pipe.put(pins[0]) if e2e_b else None
    for k, b in enumerate(e2e_b):
        nxt = pipe.put(pins[k + 1]) if k + 1 < len(e2e_b) else None
        pipe.update(staged, b["counts"], b["ex_rows"], b["new"], U_host=Uh[k % 2], v_host=vh[k % 2])
        staged = nxt
        N = b["N"]
        h2d += N * J * 8 + (b["M_old"] + b["L"]) * (8 + 4 + 1) + 8
        d2h += N * R * 8 + J * R * 8
    pipe.finish()
    e3.record(stream)
    torch.cuda.synchronize()
    state.check()
    e2e_ms = e2.elapsed_time(e3)
    if world > 1:
        tt = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e_elems = sum(b["N"] for b in e2e_b) * J
    if world > 1:
        te = torch.tensor([e2e_elems], device=dev, dtype=torch.float64)
        dist.all_reduce(te)
        e2e_elems = float(te.item())
    e2e_value = e2e_elems / (e2e_ms / 1e3) if e2e_b else None

    # the drop-in API a reference user calls: StreamState.update(UpdateBatch)
    # with host batches of per-slice numpy arrays (gather into pinned memory,
    # H2D, update, sync + SolveError check, v_used read back), like the
    # reference's update() whose `seconds` include its staging (rank 0, N=1)
    dropin = None
    if world == 1 and args.dropin_steps > 0:
        dropin = run_dropin(cfg, arrays, args.dropin_steps, dev)
    parity = None
    if world == 1 and args.parity_steps > 0:
        parity = run_parity(cfg, args.parity_steps, dev)
    als = None
    if world == 1 and args.als:
        als = {name: als_timing(name, dev) for name in ("medium", "daily")}

    # roofline of the dominant kernel
    phase_ms = {nat.PHASES[i]: ms_arr[i] for i in range(nph)}
    phase_n = {nat.PHASES[i]: cnt_arr[i] for i in range(nph)}
    dom = max(phase_ms, key=lambda k: phase_ms[k])
    nb = len(profiled)
    nt = len(timed)
    N_avg = sum(b["N"] for b in timed) / nt
    M_old_avg = sum(b["M_old"] for b in timed) / nt
    L_avg = sum(b["L"] for b in timed) / nt
    nsplit = torch.cuda.get_device_properties(dev).multi_processor_count  # streaming GEMM: one slot per CTA
    peak, peak_kind = peaks()
    per_launch_ms = phase_ms[dom] / max(phase_n[dom], 1)
    stt = batch_stats(profiled)
    bigx = bool(L.dash_ctx_path_flags(state._ctx) & nat.PATH_BIGX)
    kb = kernel_bytes(dom, stt, J, R, nsplit, bigx=bigx)
    per_kernel = {}
    for ph in phase_ms:
        if phase_n[ph]:
            ms1 = phase_ms[ph] / phase_n[ph]
            kb1 = kernel_bytes(ph, stt, J, R, nsplit, bigx=bigx)
            kf1 = kernel_flops(ph, stt, J, R, bigx=bigx)
            per_kernel[ph] = {"ms_per_launch": ms1, "alg_bytes": kb1,
                              "gbs": kb1 / (ms1 / 1e3) / 1e9 if kb1 else None,
                              "frac_hbm": kb1 / (ms1 / 1e3) / 1e9 / peak if kb1 else None}
            if kf1:
                per_kernel[ph].update({"alg_flops": kf1, "tflops": kf1 / (ms1 / 1e3) / 1e12,
                                       "frac_fp64_tensor": kf1 / (ms1 / 1e3) / 1e12 / FP64_TENSOR_PEAK})
    achieved = kb / (per_launch_ms / 1e3) / 1e9
    step_bytes = algorithmic_bytes(N_avg, J, R, M_old_avg, L_avg)
    step_achieved = step_bytes / (ms_per_step / 1e3) / 1e9

    out = None
    if rank == 0:
        out = {
            "metric": f"X elements/s of the DASH update step ({cfg.name} stream, FP64)",
            "value": value, "unit": "elements/s", "n_gpus": world, "steps": len(timed),
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (planted low-rank + N(0,0.1) noise, drawn on device; planted initial state)",
            "config": workload_config(cfg, sched, args.warmup, args.warmup + args.steps, f"slice-sharded x{world}"),
            "roofline": roofline_of(dom, per_kernel, achieved, peak, peak_kind, per_launch_ms, kb, cfg.name),
            "step_roofline": {"alg_bytes": step_bytes, "achieved_gbs": step_achieved,
                              "frac": step_achieved / peak,
                              "alg_flops": algorithmic_flops(N_avg, J, R, M_old_avg + L_avg),
                              "tflops": algorithmic_flops(N_avg, J, R, M_old_avg + L_avg) / (ms_per_step / 1e3) / 1e12},
            "phase_ms_per_step": {k: v / nb for k, v in phase_ms.items() if phase_n[k]},
            "per_kernel_roofline": per_kernel,
            "e2e": {"value": e2e_value, "unit": "elements/s", "h2d_bytes_per_step": h2d / max(len(e2e_b), 1),
                    "d2h_bytes_per_step": d2h / max(len(e2e_b), 1),
                    "ms_per_step": e2e_ms / max(len(e2e_b), 1), "steps": len(e2e_b)},
            "gpu_launches": launches,
            "lu_fallbacks": fallbacks,
            "fp32": fp32,
            "e2e_dropin": dropin,
            "parity": parity,
            "fitness": fitness,
            "als": als,
            "clocks": clocks,
        }
    del batches
    if world > 1:
        dist.barrier()
    return out, cfg


def run_dropin(cfg, arrays, steps, dev):
    """e2e through StreamState.update(UpdateBatch) on host batches (the
    reference's call): wall time per update, synchronous like the reference."""
    import torch

    from paper_2305_18376_b200.stream import StreamState
    st = StreamState.from_arrays(arrays, device=dev)
    hb, gen = host_stream(cfg, steps + 1, seed_extra=1)
    del hb
    batches = [(b, N) for b, N in gen()]
    st.reserve_u_history(sum(N for _, N in batches))
    st.update(batches[0][0])  # warm-up (pinned staging buffers, thread pool)
    torch.cuda.synchronize()
    times, elems, h2d, d2h = [], 0, 0, 0
    for b, N in batches[1:]:
        t0 = time.perf_counter()
        st.update(b)
        times.append(time.perf_counter() - t0)
        elems += N * cfg.J
        h2d += N * cfg.J * 8 + (b.slice_count) * 13 + 8
        d2h += cfg.J * cfg.R * 8 + 8
    secs = sum(times)
    return {"value": elems / secs, "unit": "elements/s", "ms_per_step": 1e3 * secs / len(times),
            "steps": len(times), "h2d_bytes_per_step": h2d / len(times), "d2h_bytes_per_step": d2h / len(times),
            "api": "StreamState.update(UpdateBatch) with host numpy rows (wall clock, synchronous)"}


def run_parity(cfg, steps, dev):
    """Parity of the timed configuration at its full size (the oracle as the
    checker, outside every timed region): `steps` updates of this config
    through StreamState.update on a fresh planted state (FP64, and the FP32
    data mode), each compared with the CPU oracle on the same host batches --
    max over the updates of max|a - b| / max|b| per array."""
    import torch

    from oracle import dash_oracle as orc
    from paper_2305_18376_b200.evaluate import local_error
    from paper_2305_18376_b200.stream import StreamState
    orc.build_c()
    arrays, gen = host_stream(cfg, steps, seed_extra=2)
    gpu = StreamState.from_arrays(arrays, device=dev)
    g32 = StreamState.from_arrays(arrays, device=dev, dtype=torch.float32)
    cpu = oracle_state(arrays)

    def rel(a, b):
        return float(np.abs(np.asarray(a) - b).max() / max(float(np.abs(b).max()), 1e-300))

    worst, worst32 = {}, {}
    for batch, _ in gen():
        ids = [sid for sid, _, _ in batch.items()]
        res, r32, ref = gpu.update(batch), g32.update(batch), cpu.update(batch)
        Uo = np.concatenate([ref["u_new"][s] for s in ids])
        w_rows = {s: cpu.W[cpu.row_of(s)] for s in ids}
        le_ref = orc.local_error([(s, r) for s, r, _ in batch.items()], ref["u_new"], w_rows, cpu.V)[0]
        for eng, r, acc in ((gpu, res, worst), (g32, r32, worst32)):
            errs = {"u_new": rel(r.u_new.device_tensor.cpu().numpy(), Uo), "v_used": rel(r.v_used, ref["v_used"])}
            for name in ("W", "C", "D", "F", "G", "V"):
                errs[name] = rel(getattr(eng, name), getattr(cpu, name))
            le = local_error([(s, r_) for s, r_, _ in batch.items()], r.u_new, eng)[0]
            errs["local_error"] = abs(le - le_ref) / max(abs(le_ref), 1e-300)
            for k, v in errs.items():
                acc[k] = max(acc.get(k, 0.0), v)
    return {"updates": steps, "config": cfg.name, "K0": cfg.K0, "against": "CPU oracle (oracle/dash_oracle.py), same host batches",
            "metric": "max over updates of max|gpu - oracle| / max|oracle| per array",
            "fp64": {"tol": 1e-8, "max_err": worst, "ok": bool(max(worst.values()) <= 1e-8)},
            "fp32_data_mode": {"tol": 1e-3, "max_err": worst32, "ok": bool(max(worst32.values()) <= 1e-3)}}


def als_timing(name, dev, iters=10):
    """One parafac2_als sweep at a BASELINE shape (initialize's fit and the
    baseline refit, tol=0 so every sweep runs), on a device-resident tensor of
    that shape drawn from the planted generator; SURVEY 8(d) ALS roofline:
    >= 2 x 8 x sum(I_k) x J bytes per sweep (target and projection passes)."""
    import torch

    from paper_2305_18376_b200 import workloads as wl
    from paper_2305_18376_b200.als import parafac2_als
    from paper_2305_18376_b200.history import DeviceTensor
    cfg = wl.CONFIGS[name]
    sch = wl.make_schedule(cfg)
    counts = sch.init_len.astype(np.int64)
    row_ptr = np.zeros(len(counts) + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    N, J, R = int(row_ptr[-1]), cfg.J, cfg.R
    H, V = wl.true_factors(cfg)
    g = torch.Generator(device=dev)
    g.manual_seed(cfg.seed)
    scale = torch.as_tensor(np.repeat(1.0 / np.sqrt(counts), counts), device=dev)
    w = torch.rand((len(counts), R), generator=g, device=dev, dtype=torch.float64)
    q = torch.randn((N, R), generator=g, device=dev, dtype=torch.float64) * scale[:, None]
    rows_of = torch.as_tensor(np.repeat(np.arange(len(counts)), counts), device=dev)
    X = ((q @ torch.as_tensor(H, device=dev)) * w[rows_of]) @ torch.as_tensor(V, device=dev).T
    X += 0.1 * torch.randn((N, J), generator=g, device=dev, dtype=torch.float64)
    del q, rows_of, scale
    dt = DeviceTensor([wl.slice_id(k) for k in range(len(counts))], row_ptr, X)
    parafac2_als(dt, R, iters=1, seed=0, tol=0.0)  # warm-up
    torch.cuda.synchronize()
    fit = []
    for n in (1, 1 + iters):  # per sweep = the difference: fit setup / host factor copies cancel
        t0 = time.perf_counter()
        parafac2_als(dt, R, iters=n, seed=1, tol=0.0)
        torch.cuda.synchronize()
        fit.append(time.perf_counter() - t0)
    sweep = (fit[1] - fit[0]) / iters
    by = 2 * 8 * N * J
    peak, _ = peaks()
    ref = ROOT / "tests" / "golden" / f"als_{name}.npz"
    ref_sweep = None
    if ref.exists():  # the reference's own 10-sweep fit of this shape, timed when the fixture was made
        with np.load(ref) as g:
            ref_sweep = 1e3 * float(g["fit_seconds"]) / len(g["losses"])
    return {"slices": len(counts), "rows": N, "J": J, "R": R, "sweep_ms": 1e3 * sweep,
            "alg_bytes_per_sweep": by, "achieved_gbs": by / sweep / 1e9, "frac_hbm": by / sweep / 1e9 / peak,
            "reference_cpu_sweep_ms": ref_sweep,
            "reference_cpu_note": "p2stream parafac2_als (numpy/OpenBLAS, 8 cores of the build container), "
                                  "fit time / sweeps, from tests/golden/make_golden_als.py",
            "fit_ms_1_sweep": 1e3 * fit[0],
            "note": "per sweep = (fit with 1 + n sweeps - fit with 1 sweep) / n, wall clock incl. the per-sweep "
                    "loss read-back for the early-exit test; fit_ms_1_sweep adds setup and the host factor copies"}


def run_fp32_arm(args, arrays, batches, dev, stream, world, J, R, prof_steps, barrier):
    """FP32 data mode: X in / U_new out in FP32 (dash_update_f32); state and
    arithmetic FP64.  Same batches (rounded), same step protocol as the FP64
    arm: W warm-ups, K device-timed steps, the profiled steps untimed (the
    stream must see every batch), then the e2e steps through HostPipeline."""
    import torch
    import torch.distributed as dist

    from paper_2305_18376_b200.distributed import ShardedStream
    from paper_2305_18376_b200.stream import HostPipeline, StreamState
    st32 = StreamState.from_arrays(arrays, device=dev, dtype=torch.float32)
    st32.reserve_u_history(sum(b["N"] for b in batches))
    eng = ShardedStream(st32, rank=int(os.environ.get("RANK", "0")), world=world) if world > 1 else st32
    X32 = [b["X"].float() for b in batches]

    def step(k):
        b = batches[k]
        return eng.update_packed(X32[k], b["counts"], b["ex_rows"], b["new"])

    W, K = args.warmup, args.steps
    for k in range(W):
        step(k)
    torch.cuda.synchronize()
    st32.check()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(W, W + K):
        step(k)
    e1.record(stream)
    torch.cuda.synchronize()
    t_ms = e0.elapsed_time(e1)
    import ctypes
    from paper_2305_18376_b200 import _native as nat
    L = nat.lib()
    L.dash_ctx_set_profiling(st32._ctx, 1)
    for k in range(W + K, W + K + prof_steps):
        step(k)
    torch.cuda.synchronize()
    nph = len(nat.PHASES)
    ms_arr = (ctypes.c_double * nph)()
    cnt_arr = (ctypes.c_int32 * nph)()
    L.dash_ctx_phase_ms(st32._ctx, ms_arr, cnt_arr, nph)
    L.dash_ctx_set_profiling(st32._ctx, 0)
    phase = {nat.PHASES[i]: ms_arr[i] / prof_steps for i in range(nph) if cnt_arr[i]}
    e2e_ks = list(range(W + K + prof_steps, len(batches)))
    pins = []
    for k in e2e_ks:
        pins.append(X32[k].cpu().pin_memory())
    maxN = max((batches[k]["N"] for k in e2e_ks), default=1)
    Uh = [torch.empty((maxN, R), dtype=torch.float32).pin_memory() for _ in range(2)]
    vh = [torch.empty((J, R), dtype=torch.float64).pin_memory() for _ in range(2)]
    pipe = HostPipeline(eng, maxN, J, device=dev)
    torch.cuda.synchronize()
    st32.check()
    barrier()
    h2d = d2h = 0
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    pipe.start()
    staged = pipe.put(pins[0]) if e2e_ks else None
    for i, k in enumerate(e2e_ks):
        b = batches[k]
        nxt = pipe.put(pins[i + 1]) if i + 1 < len(e2e_ks) else None
        pipe.update(staged, b["counts"], b["ex_rows"], b["new"], U_host=Uh[i % 2], v_host=vh[i % 2])
        staged = nxt
        h2d += b["N"] * J * 4 + (b["M_old"] + b["L"]) * (8 + 4 + 1) + 8
        d2h += b["N"] * R * 4 + J * R * 8
    pipe.finish()
    e3.record(stream)
    torch.cuda.synchronize()
    st32.check()
    e2e_ms = e2.elapsed_time(e3)
    elems = sum(batches[k]["N"] for k in range(W, W + K)) * J
    e2e_elems = sum(batches[k]["N"] for k in e2e_ks) * J
    vals = torch.tensor([t_ms, e2e_ms, elems, e2e_elems], device=dev, dtype=torch.float64)
    if world > 1:
        mx = vals[:2].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = vals[2:].clone()
        dist.all_reduce(sm)
        vals = torch.cat([mx, sm])
    t_ms, e2e_ms, elems, e2e_elems = (float(v) for v in vals.tolist())
    del X32, pins
    N_avg = sum(batches[k]["N"] for k in range(W, W + K)) / K
    M_old = sum(batches[k]["M_old"] for k in range(W, W + K)) / K
    L_avg = sum(batches[k]["L"] for k in range(W, W + K)) / K
    # algorithmic bytes with FP32 X and U_new (state terms stay FP64)
    by = 4 * (N_avg * J + N_avg * R) + 8 * (2 * M_old * (R * R + 2 * R) + L_avg * (R * R + 2 * R)
                                             + 3 * J * R + 2 * R * R)
    peak, _ = peaks()
    ms = t_ms / K
    return {"dtype": "f32 data (X in, U_new out); f64 state and arithmetic",
            "value": elems / (t_ms / 1e3), "unit": "elements/s", "ms_per_step": ms, "steps": K,
            "step_roofline": {"alg_bytes": by, "achieved_gbs": by / (ms / 1e3) / 1e9,
                              "frac": by / (ms / 1e3) / 1e9 / peak},
            "phase_ms_per_step": phase,
            "e2e": {"value": e2e_elems / (e2e_ms / 1e3) if e2e_ks else None, "unit": "elements/s",
                    "h2d_bytes_per_step": h2d / max(len(e2e_ks), 1),
                    "d2h_bytes_per_step": d2h / max(len(e2e_ks), 1),
                    "ms_per_step": e2e_ms / max(len(e2e_ks), 1), "steps": len(e2e_ks)},
            "parity": "tests/test_gpu_fp32.py: <= 1e-3 vs the FP64 oracle, <= 1e-5 vs the oracle on FP32-rounded X"}


# ---------------------------------------------------------------------------
# CPU arms (oracle port of the reference)
# ---------------------------------------------------------------------------
def host_stream(cfg, steps, seed_extra=0):
    """Planted state + host batches for the CPU reference (same law as the
    device generator)."""
    from paper_2305_18376_b200 import workloads as wl
    from paper_2305_18376_b200.tensor import NewSlice, UpdateBatch
    sched = Schedule(cfg, steps, cfg.seed)
    H, V = wl.true_factors(cfg)
    R, J = cfg.R, cfg.J
    n_all = cfg.K0 + sum(len(n) for n in sched.new_len)
    w_true = np.random.default_rng([cfg.seed, 12]).uniform(size=(n_all, R))
    D0 = H.T @ H
    vtv = V.T @ V
    W0 = w_true[:cfg.K0]
    G0 = np.einsum("kr,rz,kz->rz", W0, D0, W0)
    G0 = (G0 + G0.T) / 2.0
    arrays = {"slice_ids": [wl.slice_id(k) for k in range(cfg.K0)], "W": W0, "V": V,
              "C": np.einsum("rz,kz,zr->kr", D0, W0, vtv),
              "D": np.broadcast_to(D0, (cfg.K0, R, R)).copy(), "F": V @ G0, "G": G0,
              "forgetting": cfg.forgetting}
    rng = np.random.default_rng([cfg.seed, 13, seed_extra])

    def batches():
        active = cfg.K0
        for t in range(steps):
            add = sched.adds[t]
            new = sched.new_len[t]
            counts = np.concatenate([add, new])
            N = int(counts.sum())
            ks = np.repeat(np.arange(active + len(new)), counts)
            q = rng.standard_normal((N, R)) / np.sqrt(1100.0)
            X = ((q @ H) * w_true[ks]) @ V.T + 0.1 * rng.standard_normal((N, J))
            offs = np.concatenate([[0], np.cumsum(counts)])
            existing = {wl.slice_id(k): X[offs[k]:offs[k + 1]] for k in range(active)}
            fresh = [NewSlice(wl.slice_id(active + i), X[offs[active + i]:offs[active + i + 1]], t + 1)
                     for i in range(len(new))]
            active += len(new)
            yield UpdateBatch(t + 1, existing, fresh, (t + 1, t + 1)), N
    return arrays, batches


def oracle_state(arrays):
    from oracle import dash_oracle as orc
    R = arrays["V"].shape[1]
    return orc.OracleStreamState(arrays["slice_ids"], {s: [] for s in arrays["slice_ids"]},
                                 arrays["W"], arrays["V"], arrays["C"], arrays["D"], arrays["F"],
                                 arrays["G"], arrays["forgetting"])


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max([i.get("num_threads", 1) for i in info] or [1])
    except Exception:
        return 1


def time_oracle(cfg, warm, steps):
    """Time the CPU oracle on `steps` full updates after `warm` warm-ups."""
    from oracle import dash_oracle as orc
    orc.build_c()
    arrays, gen = host_stream(cfg, warm + steps)
    st = oracle_state(arrays)
    times, elems = [], 0
    for t, (batch, N) in enumerate(gen()):
        t0 = time.perf_counter()
        st.update(batch)
        dt = time.perf_counter() - t0
        if t >= warm:
            times.append(dt)
            elems += N * cfg.J
    return elems, sum(times), len(times)


def cpu_baseline(cfg, steps):
    elems, secs, n = time_oracle(cfg, 1, steps)
    return {"value": elems / secs, "unit": "elements/s", "cores": blas_threads(), "kind": "port",
            "sample": f"{n} full {cfg.name} updates after 1 warm-up (oracle: numpy/OpenBLAS + C port of "
                      f"the numba group_update; the per-slice kernel is single-threaded, BLAS uses "
                      f"{blas_threads()} threads); {secs:.1f} s of CPU work",
            "ms_per_step": 1e3 * secs / n}


def run_reference(args):
    from paper_2305_18376_b200 import workloads as wl
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    cfg = wl.CONFIGS[args.config]
    if args.K0:
        cfg = wl.scaled(cfg, K0=args.K0)
    elems, secs, n = time_oracle(cfg, args.warmup, args.steps)
    value = elems / secs
    cores = blas_threads()
    return {
        "metric": f"X elements/s of the DASH update step ({cfg.name} stream, FP64)",
        "value": value, "unit": "elements/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": n, "warmup": args.warmup, "ms_per_step": 1e3 * secs / n,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (planted low-rank + N(0,0.1) noise, host numpy)",
        "config": workload_config(cfg, Schedule(cfg, args.warmup + args.steps, cfg.seed), args.warmup,
                                  args.warmup + args.steps, f"slice-sharded x{int(os.environ.get('WORLD_SIZE', '1'))}"),
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "elements/s", "cores": cores, "kind": "port",
                         "sample": f"{n} full {cfg.name} updates of the oracle port of p2stream "
                                   f"StreamState.update (numpy/OpenBLAS {cores} threads + C port of the "
                                   f"numba kernel, single-threaded)"},
        "e2e": {"value": value, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    args = parse()
    if args.impl == "reference":
        out = run_reference(args)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    out, cfg = run_gpu(args)
    if out is not None:
        world = out["n_gpus"]
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(cfg, args.cpu_steps)
        else:
            out["cpu_baseline"] = None
        print(json.dumps(out), flush=True)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
