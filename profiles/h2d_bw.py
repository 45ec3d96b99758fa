"""Pinned host<->device copy bandwidth on this box (what bounds the e2e
numbers: 252 MB H2D + 25 MB D2H per config-2 frame)."""
import json

import torch

out = {}
for mb in (6, 53, 199):
    n = mb * (1 << 20) // 4
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                     ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        out[f"{name}_{mb}MB_GBps"] = round(n * 4 / ms / 1e6, 1)
print(json.dumps(out))
