"""Host-ABI frame throughput on config 2: synchronous lvsg_forward_render
versus pipelined lvsg_submit_frame / lvsg_wait_frame (two in flight), over
N frames with pinned buffers. Prints one JSON line (ms per frame)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(n=20):
    import torch
    import paper_2411_16680_b200 as q
    from paper_2411_16680_b200 import workloads as wl
    case = wl.config2()
    m = q.Model(case.cfg, device=0)
    m.init_weights(case.seed)
    pin = lambda a: torch.from_numpy(a).pin_memory()  # noqa: E731
    enc_t, ren_t = pin(case.enc_images), pin(case.ren_images)
    enc, ren = enc_t.numpy(), ren_t.numpy()
    plan = q.plan_forward(case.cfg, enc.shape[1], enc.shape[2])
    out_t = [torch.empty((plan.out_height, plan.out_width, 3)).pin_memory() for _ in range(2)]
    outs = [o.numpy() for o in out_t]
    res = {}
    for _ in range(2):
        m.forward_render(enc, case.enc_cams, ren, case.ren_cams, case.target, out=outs[0])
    t0 = time.perf_counter()
    for _ in range(n):
        m.forward_render(enc, case.enc_cams, ren, case.ren_cams, case.target, out=outs[0])
    res["sync_ms"] = (time.perf_counter() - t0) / n * 1e3
    pend = []
    t0 = time.perf_counter()
    for i in range(n):
        if len(pend) == 2:
            m.wait_frame(pend.pop(0))
        pend.append(m.submit_frame(enc, case.enc_cams, ren, case.ren_cams, case.target, outs[i % 2]))
    while pend:
        m.wait_frame(pend.pop(0))
    res["pipelined_ms"] = (time.perf_counter() - t0) / n * 1e3
    # submit-side host time alone (how long a submit blocks)
    ts = []
    for i in range(6):
        a = time.perf_counter()
        pend.append(m.submit_frame(enc, case.enc_cams, ren, case.ren_cams, case.target, outs[i % 2]))
        ts.append((time.perf_counter() - a) * 1e3)
        if len(pend) == 2:
            m.wait_frame(pend.pop(0))
    while pend:
        m.wait_frame(pend.pop(0))
    res["submit_host_ms"] = ts
    print(json.dumps(res))
    m.close()


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def sharded(n=10):
    """The bench's view-sharded e2e step at N=1, timed part by part."""
    import torch
    import paper_2411_16680_b200 as q
    from paper_2411_16680_b200 import workloads as wl
    dev = torch.device("cuda", 0)
    case = wl.config2()
    M = case.cfg.views
    m = q.Model(case.cfg, device=0)
    m.init_weights(case.seed)
    enc_h = torch.from_numpy(case.enc_images).pin_memory()
    ren_h = torch.from_numpy(case.ren_images).pin_memory()
    enc = enc_h.to(dev)
    He, We = enc.shape[1], enc.shape[2]
    plan = q.plan_forward(case.cfg, He, We)
    out = torch.empty((plan.out_height, plan.out_width, 3)).pin_memory().numpy()
    r_np = ren_h.numpy()
    st = torch.cuda.Stream(device=dev)
    parts = {"copy": 0.0, "encode": 0.0, "sync": 0.0, "forward_render_null": 0.0}
    for i in range(n + 2):
        a = time.perf_counter()
        with torch.cuda.stream(st):
            enc.copy_(enc_h, non_blocking=True)
            b = time.perf_counter()
            m.encode_device(enc, 0, M, st)
        c = time.perf_counter()
        st.synchronize()
        d = time.perf_counter()
        m.forward_render(None, case.enc_cams, r_np, case.ren_cams, case.target, out=out,
                         enc_hw=(He, We))
        e = time.perf_counter()
        if i >= 2:
            for k, v in zip(parts, (b - a, c - b, d - c, e - d)):
                parts[k] += v * 1e3 / n
    print(json.dumps({"sharded_parts_ms": parts}))
    m.close()


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "sharded":
    sharded()
