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
    """SIMT (impl 1) and the tcgen05 conv (impl 2; falls back to SIMT off the
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
        # fp32-accurate: the 3-term tensor-core split keeps ~2^-22 relative per product
        assert err <= 2e-5 * max(1.0, scale), (impl, err)


def _gelu(x):
    from scipy.special import erf
    return 0.5 * x * (1.0 + erf(x / np.sqrt(2.0)))


@pytest.mark.parametrize("impl", [1, 2])
@pytest.mark.parametrize("variant", ["rms_gelu", "slice_resid", "strided"])
def test_conv3x3_fused_options(oracle, model, impl, variant):
    """The fused conv options the solve uses: rms-norm input + GELU
    (conv_mlp_residual), weight-channel slices accumulated through the
    residual (the split update-CNN stem), and a padded pixel stride (the
    feedback rows), against an f64 NumPy restatement."""
    import torch
    rng = np.random.default_rng(11)
    B, H, W, C = 2, 19, 29, 32
    dev = torch.device("cuda:0")
    x = rng.standard_normal((B, H, W, 36)).astype(np.float32)
    w = (rng.standard_normal((C, 97, 3, 3)) / np.sqrt(9 * 97)).astype(np.float32)
    bias = rng.standard_normal(C).astype(np.float32)
    gain = rng.uniform(0.5, 1.5, C).astype(np.float32)
    res = rng.standard_normal((B, H, W, C)).astype(np.float32)
    xd = x.astype(np.float64)

    def conv(inp, wk):  # inp [B,H,W,Cin] f64, wk [C, Cin, 3, 3]
        p = np.pad(inp, ((0, 0), (1, 1), (1, 1), (0, 0)))
        out = np.zeros((B, H, W, C))
        for dy in range(3):
            for dx in range(3):
                out += np.einsum("bhwc,oc->bhwo", p[:, dy:dy + H, dx:dx + W], wk[:, :, dy, dx])
        return out

    y = torch.empty((B, H, W, C), dtype=torch.float32, device=dev)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    if variant == "rms_gelu":
        xs = np.ascontiguousarray(x[..., :C])
        n = xs.astype(np.float64) / np.sqrt((xs.astype(np.float64) ** 2).mean(-1, keepdims=True) + 1e-6)
        wk = np.ascontiguousarray(w[:, :C])
        want = _gelu(conv(n * gain, wk.astype(np.float64)) + bias)
        model.stage_conv3x3_fused(t(xs), t(wk), t(bias), y, C, norm_gain_t=t(gain), gelu=True,
                                  impl=impl)
    elif variant == "slice_resid":
        xs = np.ascontiguousarray(x[..., :C])
        want = res + conv(xd[..., :C], w[:, 33:65].astype(np.float64))
        y.copy_(t(res))
        model.stage_conv3x3_fused(t(xs), t(w), None, y, C, ci0=33, resid_t=y, impl=impl)
    else:
        want = conv(xd[..., :C], w[:, 0:32].astype(np.float64)) + bias
        model.stage_conv3x3_fused(t(x), t(w), t(bias), y, C, ci0=0, impl=impl)
    got = y.cpu().numpy()
    err = np.abs(got - want).max()
    assert err <= 3e-5 * max(1.0, np.abs(want).max()), (variant, impl, err)


@pytest.mark.parametrize("where", ["input", "weight"])
def test_fp16_split_overflow_is_numeric_error(model, where):
    """The tensor-core conv's 3-term fp16 split cannot hold |x| >= 65520 (the
    hi term rounds to inf): such an operand reports NumericError instead of a
    silently wrong result; the SIMT conv (impl 1) computes it in fp32, and the
    context stays usable."""
    import torch
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(5)
    x = rng.standard_normal((1, 16, 16, 32)).astype(np.float32)
    w = (rng.standard_normal((32, 32, 3, 3)) / 17.0).astype(np.float32)
    if where == "input":
        x[0, 5, 7, 3] = 1.0e5
    else:
        w[4, 9, 1, 1] = -7.0e4
    y = torch.empty((1, 16, 16, 32), dtype=torch.float32, device=dev)
    t = lambda a: torch.from_numpy(a).to(dev)  # noqa: E731
    with pytest.raises(q.NumericError):
        model.stage_conv3x3(t(x), t(w), None, y, impl=2)
    model.stage_conv3x3(t(x), t(w), None, y, impl=1)  # fp32 SIMT: fine
    assert torch.isfinite(y).all()
    x[0, 5, 7, 3] = 0.5
    w[4, 9, 1, 1] = 0.1
    model.stage_conv3x3(t(x), t(w), None, y, impl=2)  # the context recovers
    assert torch.isfinite(y).all()


def test_attention_split_overflow_is_numeric_error():
    """The same guard in the tensor-core attention: a V row whose rms-normed
    value or a head with |x| >= 65520 in the split operand -> NumericError."""
    import torch
    from cases import config1
    m = q.Model(config1().cfg, device=0)
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(6)
    P_, C, M, H = 4096, 32, 8, 1
    V = rng.standard_normal((P_, C)).astype(np.float32)
    D = rng.standard_normal((P_, M, C)).astype(np.float32)
    wq = (rng.standard_normal((H, C, C)) / np.sqrt(C)).astype(np.float32)
    wo = (rng.standard_normal((H * C, C)) / np.sqrt(C)).astype(np.float32)
    g = np.ones(C, np.float32)
    D[100, 3, :] = 2.0e5  # heads are convex mixes of Δ: this texel's head overflows
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    with pytest.raises(q.NumericError):
        m.stage_attend(t(V), t(D), t(wq), t(wo), t(g))
    D[100, 3, :] = 0.25
    Vt = t(V)
    m.stage_attend(Vt, t(D), t(wq), t(wo), t(g))
    assert torch.isfinite(Vt).all()
