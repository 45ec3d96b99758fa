"""Debug: the stage attention (heads, M) on random inputs, repeated; where
(which 128-texel tiles / CTAs / tile order) the result departs from the
oracle."""
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
CFGS = [(2, 4, 6 * 144 * 256), (2, 4, 148 * 128 * 3), (4, 4, 6 * 144 * 256), (2, 2, 6 * 144 * 256), (2, 8, 6 * 144 * 256), (1, 4, 6 * 144 * 256)]
if os.environ.get('ONLY24'): CFGS = CFGS[:1] + [(4, 4, 6 * 144 * 256), (4, 2, 6 * 144 * 256), (2, 3, 6 * 144 * 256)]
for heads, M, P_ in CFGS:
    rng = np.random.default_rng(heads * 100 + M)
    V = rng.standard_normal((P_, C)).astype(np.float32)
    D = rng.standard_normal((P_, M, C)).astype(np.float32)
    D[rng.random((P_, M)) < 0.2] = 0.0
    wq = (rng.standard_normal((heads, C, C)) / np.sqrt(C)).astype(np.float32)
    wo = (rng.standard_normal((heads * C, C)) / np.sqrt(heads * C)).astype(np.float32)
    g = (1.0 + 0.1 * rng.standard_normal(C)).astype(np.float32)
    want = o.attend_residual(V, D, wq, wo, g, False)
    m = q.Model(case.cfg, device=0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to("cuda:0")
    for rep in range(int(os.environ.get('REPS', '4'))):
        Vt = t(V)
        m.stage_attend(Vt, t(D), t(wq), t(wo), t(g))
        got = Vt.cpu().numpy()
        e = np.abs(got - want).max(1)
        bad = np.nonzero(e > 1e-4)[0]
        tiles = np.unique(bad // 128)
        ntiles = (P_ + 127) // 128
        print(f"h={heads} M={M} P={P_} rep {rep}: max {e.max():.2e}, bad texels {len(bad)}, "
              f"bad tiles {len(tiles)} of {ntiles}: {tiles[:12].tolist()} "
              f"(tile % 148: {(tiles % 148)[:12].tolist()}, order in CTA: {(tiles // 148)[:12].tolist()}; "
              f"rows in tile: {np.unique(bad % 128)[:8].tolist()})", flush=True)
    m.close()
