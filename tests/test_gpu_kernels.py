"""Per-kernel GPU checks through the C ABI stage entry points."""
import numpy as np
import pytest

import paper_2411_16680_b200 as q
from cases import nano

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def model():
    return q.Model(nano().cfg, device=0)


@pytest.mark.parametrize("B,H,W,Cin,Cout", [(2, 37, 53, 32, 32), (1, 16, 8, 32, 32),
                                            (3, 9, 15, 32, 32), (2, 20, 30, 3, 32),
                                            (1, 18, 22, 97, 32), (1, 7, 9, 8, 8)])
@pytest.mark.parametrize("impl", [1, 2])
def test_conv3x3_matches_oracle(oracle, model, B, H, W, Cin, Cout, impl):
    """SIMT (impl 1) and tcgen05 3xTF32 (impl 2; falls back to SIMT off its
    Cin = Cout = 32 shape) against the oracle conv (kernels_ref.hpp:72-96)."""
    import torch
    rng = np.random.default_rng(H * 100 + W)
    x = rng.standard_normal((B, H, W, Cin)).astype(np.float32)
    w = (rng.standard_normal((Cout, Cin, 3, 3)) / np.sqrt(9 * Cin)).astype(np.float32)
    b = rng.standard_normal(Cout).astype(np.float32)
    dev = torch.device("cuda:0")
    y = torch.empty((B, H, W, Cout), dtype=torch.float32, device=dev)
    model.stage_conv3x3(torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev),
                        torch.from_numpy(b).to(dev), y, impl=impl)
    got = y.cpu().numpy()
    for bi in range(B):
        want = oracle.conv3x3(np.ascontiguousarray(x[bi].transpose(2, 0, 1)), w, b)
        err = np.abs(got[bi].transpose(2, 0, 1) - want).max()
        scale = np.abs(want).max()
        # fp32-accurate: 3xTF32 keeps ~2^-21 relative per product
        assert err <= 2e-5 * max(1.0, scale), (impl, err)
