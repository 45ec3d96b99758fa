"""The checked build (-DLVSG_CHECKED=1): every gather tap, splat bin and run,
splat payload row and render tap is bounds-checked on the device (a failed
check prints and traps). compute-sanitizer is closed on this GPU pool, so this
is the memcheck of the index work: the whole path runs clean on several
configs and gives bit-identical frames to the default build."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "build", "variant", "checked", "liblvsg.so")

_RUN = r"""
import sys, numpy as np
sys.path[:0] = [sys.argv[1], sys.argv[1] + '/tests']
import paper_2411_16680_b200 as q
from paper_2411_16680_b200 import workloads as wl
case = {'nano': wl.nano, 'config1': wl.config1, 'c2div4': lambda: wl.config2(div=4),
        'm3div4': lambda: wl.config2(div=4, views_rig=(1, 3))}[sys.argv[2]]()
m = q.Model(case.cfg, device=0)
m.load_weights(case.store())
rgb = m.forward_render(case.enc_images, case.enc_cams, case.ren_images, case.ren_cams, case.target)
ldm = m.forward(case.enc_images, case.enc_cams, case.target, deltas=True)
out = np.empty_like(rgb)
m.wait_frame(m.submit_frame(case.enc_images, case.enc_cams, case.ren_images, case.ren_cams,
                            case.target, out))
assert np.array_equal(out.view(np.uint32), rgb.view(np.uint32))
np.save(sys.argv[3], rgb)
np.save(sys.argv[3] + '.deltas.npy', ldm.deltas)
m.close()
"""


def _sources_mtime():
    src = os.path.join(ROOT, "paper_2411_16680_b200", "csrc")
    return max(os.path.getmtime(os.path.join(src, f)) for f in os.listdir(src))


@pytest.fixture(scope="module")
def checked_lib():
    if not os.path.exists(CHECKED) or os.path.getmtime(CHECKED) < _sources_mtime():
        subprocess.run(["bash", os.path.join(ROOT, "profiles", "debug", "build_variant.sh"),
                        "checked", "-DLVSG_CHECKED=1"], cwd=ROOT, check=True, timeout=1200,
                       capture_output=True)
    return CHECKED


@pytest.mark.parametrize("name", ["nano", "config1", "c2div4", "m3div4"])
def test_checked_build_runs_clean(tmp_path, checked_lib, name):
    outs = {}
    for tag, lib in (("default", None), ("checked", checked_lib)):
        env = dict(os.environ)
        env.pop("LVSG_LIB", None)
        if lib:
            env["LVSG_LIB"] = lib
        path = str(tmp_path / f"{tag}.npy")
        r = subprocess.run([sys.executable, "-c", _RUN, ROOT, name, path], env=env,
                           capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, (tag, r.stdout[-2000:] + r.stderr[-2000:])
        assert "LVSG_CHECK failed" not in r.stdout + r.stderr
        outs[tag] = (np.load(path), np.load(path + ".deltas.npy"))
    for a, b in zip(outs["default"], outs["checked"]):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
