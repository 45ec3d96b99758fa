"""Debug: attention (2, 4) -- which head's path is wrong (zero one head's Wo
block), and the bad rows of the bad tiles."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np
import torch
import paper_2411_16680_b200 as q
from bindings import Oracle
from cases import config1

o = Oracle()
case = config1()
C = 32
heads, M, P_ = 2, 4, 6 * 144 * 256
rng = np.random.default_rng(heads * 100 + M)
V = rng.standard_normal((P_, C)).astype(np.float32)
D = rng.standard_normal((P_, M, C)).astype(np.float32)
D[rng.random((P_, M)) < 0.2] = 0.0
wq = (rng.standard_normal((heads, C, C)) / np.sqrt(C)).astype(np.float32)
wo0 = (rng.standard_normal((heads * C, C)) / np.sqrt(heads * C)).astype(np.float32)
g = (1.0 + 0.1 * rng.standard_normal(C)).astype(np.float32)
m = q.Model(case.cfg, device=0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to("cuda:0")
for name, zero_head in (("both", None), ("head0 only", 1), ("head1 only", 0)):
    wo = wo0.copy()
    if zero_head is not None:
        wo[zero_head * C:(zero_head + 1) * C] = 0
    want = o.attend_residual(V, D, wq, wo, g, False)
    for rep in range(int(os.environ.get("REPS", "3"))):
        Vt = t(V)
        m.stage_attend(Vt, t(D), t(wq), t(wo), t(g))
        got = Vt.cpu().numpy()
        e = np.abs(got - want).max(1)
        bad = np.nonzero(e > 1e-4)[0]
        print(f"{name} rep {rep}: max {e.max():.2e} bad {len(bad)}: texels {bad[:16].tolist()} "
              f"rows {(bad % 128)[:16].tolist()}", flush=True)
        if len(bad):
            b0 = bad[0]
            # is the wrong V the oracle's V of a different texel, or V + O of another texel?
            d = got[b0] - V[b0]
            w = want[b0] - V[b0]
            print("   O got", np.round(d[:6], 4), "want", np.round(w[:6], 4), flush=True)
