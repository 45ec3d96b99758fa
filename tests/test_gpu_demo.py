"""forward-demo driver (paper_2411_16680_b200/demo.py, the reference's
run_forward_demo, tools/main.cpp:511-611) on the B200: outputs written, the
LDM container readable by the QNTC codec, the frame equal to the oracle's
within the parity gate, and the T_V + M * T_image fit present."""
import json
import os

import numpy as np
import pytest

from paper_2411_16680_b200 import demo, qntc
from paper_2411_16680_b200 import workloads as wl

pytestmark = pytest.mark.gpu


def test_forward_demo_outputs(tmp_path, oracle):
    res = demo.run("nano", str(tmp_path), seed=3, sweep=(2, 4), frames=3)  # nano has 4 views
    case = wl.nano()
    rgb = np.load(tmp_path / "target.npy")
    ref = oracle.forward_render(case.cfg, case.enc_images, case.enc_cams, case.ren_images,
                                case.ren_cams, case.target, case.flat(), outputs=("rgb",))["rgb"]
    assert float(np.max(np.abs(rgb - ref))) <= 1e-3
    ents = {e.name: e.array for e in qntc.unpack_tensors((tmp_path / "ldm.qntc").read_bytes())}
    L, Ho, Wo = ents["depth"].shape
    assert (Ho, Wo) == rgb.shape[:2] and ents["blend"].shape == (L, Ho, Wo, case.cfg.views)
    w = qntc.unpack_tensors((tmp_path / "weights.qntc").read_bytes())
    assert [e.name for e in w] == qntc.param_names(case.cfg)
    t = json.loads((tmp_path / "timings.json").read_text())
    assert set(t["per_view_ms"]) == {"2", "4"} and "t_image_ms" in t and "t_volume_ms" in t
    assert all(p["ms_per_frame"] > 0 and p["launches"] > 0 for p in t["per_view_ms"].values())
    assert res["views"] == case.cfg.views
