"""Times the tensor-core conv3x3 stage on the level-0 encoder shape
[8, 576, 960, 32] through the C ABI (lvsg_stage_conv3x3_fused), for the
plain / rms+gelu / residual variants. Run once per library build
(LVSG_LIB=... python profiles/conv_probe.py) to compare probe builds."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_16680_b200 as q  # noqa: E402


def main():
    B, H, W, C = 8, 576, 960, 32
    if len(sys.argv) > 1:
        B, H, W = map(int, sys.argv[1].split(","))
    dev = torch.device("cuda:0")
    m = q.Model(q.nano_config(), device=0)
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn((B, H, W, C), device=dev, generator=g)
    w = torch.randn((C, C, 3, 3), device=dev, generator=g) / 17.0
    b = torch.randn(C, device=dev, generator=g)
    gain = torch.rand(C, device=dev, generator=g) + 0.5
    res = torch.randn((B, H, W, C), device=dev, generator=g)
    y = torch.empty_like(x)
    st = torch.cuda.ExternalStream(m._lib.lvsg_stream(m._h))
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    variants = {
        "plain": dict(),
        "rms_gelu": dict(norm_gain_t=gain, gelu=True),
        "resid": dict(resid_t=res),
    }
    impl = int(os.environ.get("CONV_IMPL", "2"))
    out = {"lib": os.environ.get("LVSG_LIB", "default"), "impl": impl, "shape": [B, H, W, C]}
    for name, kw in variants.items():
        ts = []
        for it in range(8):
            flush.fill_(it)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            m.stage_conv3x3_fused(x, w, b, y, C, impl=impl, **kw)
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1000)
        tiles = B * ((H + 15) // 16) * ((W + 7) // 8)
        med = float(np.median(ts[2:]))
        out[name] = {"us": round(med, 1), "us_per_tile_per_sm": round(med / (tiles / 148), 3)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
