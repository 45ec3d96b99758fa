"""The reference-side drop-in (include/lvsg_lvs.hpp) driven by the
reference's own code: oracle/_ref/adapter_check runs lvs::forward +
render_target and the same sequence through the adapter, on the B200."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

EXE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "adapter_check")


def test_reference_adapter_drop_in():
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/adapter_check not built (reference sources absent at build)")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
