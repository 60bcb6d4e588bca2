"""Pinned host <-> device copy bandwidth on this box (the e2e ceiling)."""
import torch, time
n = 835_000_000 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
u = torch.empty(104_000_000 // 8, dtype=torch.float64, device="cuda")
uh = torch.empty_like(u, device="cpu").pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def bw(fn, nbytes, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [fn() for _ in range(reps)]; e1.record(); torch.cuda.synchronize()
    return nbytes * reps / (e0.elapsed_time(e1) / 1e3) / 1e9
print("H2D one copy   GB/s", round(bw(lambda: d.copy_(h, non_blocking=True), n * 8), 1))
print("D2H one copy   GB/s", round(bw(lambda: h.copy_(d, non_blocking=True), n * 8), 1))
def split(k):
    c = n // k
    def f():
        for i in range(k):
            st = s1 if i % 2 == 0 else s2
            with torch.cuda.stream(st):
                d[i * c:(i + 1) * c].copy_(h[i * c:(i + 1) * c], non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    return f
for k in (2, 4, 8):
    print(f"H2D {k} chunks on 2 streams GB/s", round(bw(split(k), n * 8), 1))
def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        uh.copy_(u, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
t0 = time.perf_counter(); 
print("H2D 835MB + D2H 104MB concurrent: effective H2D GB/s", round(bw(both, n * 8), 1))
