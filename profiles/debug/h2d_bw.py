"""Host<->device copy bandwidth on the GPU box: pinned H2D / D2H of the
bench's per-frame upload (252 MB) as one copy and as per-view copies, alone
and concurrent with each other."""
import time
import torch

dev = torch.device("cuda", 0)
n = 252149760 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device=dev)
o = torch.empty(24883200 // 4, dtype=torch.float32).pin_memory()
od = torch.empty_like(o, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def one():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)


def per_view():
    with torch.cuda.stream(s1):
        for v in range(8):
            a, b = v * n // 8, (v + 1) * n // 8
            d[a:b].copy_(h[a:b], non_blocking=True)


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        o.copy_(od, non_blocking=True)


for name, fn, by in (("h2d one copy", one, n * 4), ("h2d per view", per_view, n * 4),
                     ("h2d + d2h concurrent", both, n * 4)):
    t = timed(fn)
    print(f"{name}: {t * 1e3:.2f} ms, {by / t / 1e9:.1f} GB/s")
