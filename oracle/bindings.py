"""ctypes bindings for the oracle (TEST INFRASTRUCTURE ONLY).

  * `Oracle`    — oracle/liboracle.so, the C restatement (lvs_oracle.c).
  * `Reference` — oracle/_ref/libref.so, the reference library itself built
                  from /root/reference/proj with the shims (oracle/Makefile).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2411_16680_b200 import capi  # noqa: E402  (struct layouts only)

ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref.so")
REF_UNIT = os.path.join(HERE, "_ref", "lvs_unit")
REF_SRC = "/root/reference/proj"

P = ctypes.POINTER
vp = ctypes.c_void_p
i64 = ctypes.c_int64
sz = ctypes.c_size_t


def _f32(a):
    if a is None:
        return None
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(vp)


def build(ref: bool = True) -> None:
    """Builds liboracle.so and, when the reference sources are present,
    oracle/_ref (only in the build container; the GPU box gets the files)."""
    subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    if ref and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)


def _cams(cams):
    arr = (capi.CameraC * len(cams))()
    for i, c in enumerate(cams):
        arr[i] = c if isinstance(c, capi.CameraC) else c.to_c()
    return arr


def _fr(fr):
    return fr if isinstance(fr, capi.FrustumC) else fr.to_c()


class _Err:
    def __init__(self):
        self.buf = ctypes.create_string_buffer(512)

    @property
    def msg(self):
        return self.buf.value.decode(errors="replace")


class Oracle:
    def __init__(self, threads: int | None = None):
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        self.lib = ctypes.CDLL(ORACLE_SO)
        L = self.lib
        L.lvso_set_threads.argtypes = [ctypes.c_int]
        L.lvso_forward_render_ex.argtypes = [P(capi.ModelConfigC), i64, vp, i64, i64,
                                             P(capi.CameraC), vp, i64, i64, P(capi.CameraC),
                                             P(capi.FrustumC), vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                             ctypes.c_char_p, ctypes.c_size_t]
        L.lvso_world_points.argtypes = [P(capi.FrustumC), vp, i64, i64, i64, vp]
        L.lvso_footprints.argtypes = [P(capi.CameraC), vp, i64, vp, vp, vp]
        L.lvso_gather.argtypes = [P(capi.CameraC), vp, i64, i64, i64, vp, i64, vp, vp]
        L.lvso_upsample_activate.argtypes = [P(capi.FrustumC), vp, i64, i64, i64, i64, vp, vp, vp,
                                             i64, i64, i64, vp, vp, vp]
        L.lvso_render_target.argtypes = [P(capi.FrustumC), vp, vp, vp, i64, i64, i64, i64, vp,
                                         i64, i64, P(capi.CameraC), vp]
        L.lvso_conv3x3.argtypes = [vp, vp, vp, vp, i64, i64, i64, i64]
        L.lvso_trace_margins.argtypes = [ctypes.c_double, vp, i64]
        L.lvso_trace_count.restype = i64
        L.lvso_attend_residual.argtypes = [vp, vp, i64, i64, i64, i64, vp, vp, vp, ctypes.c_int]
        L.lvso_render_to_view.argtypes = [P(capi.FrustumC), vp, i64, i64, i64, i64, i64, vp, vp,
                                          vp, P(capi.CameraC), vp]
        self.set_threads(threads or os.cpu_count() or 1)

    def set_threads(self, n: int):
        self.threads = int(n)
        self.lib.lvso_set_threads(self.threads)

    def forward_render(self, cfg, enc_images, enc_cams, render_images, render_cams, target,
                       weights, plan_out=None, outputs=("rgb",)):
        """Returns a dict with the requested outputs among rgb, depth,
        density, blend, blend_logits, volume, deltas, rgb_direct."""
        return _forward_render(self.lib.lvso_forward_render_ex, cfg, enc_images, enc_cams,
                               render_images, render_cams, target, weights, outputs,
                               errfirst=False)

    def world_points(self, fr, depth):
        L_, H, W = depth.shape
        out = np.zeros((L_, H, W, 3), np.float32)
        bad = self.lib.lvso_world_points(ctypes.byref(_fr(fr)), _f32(depth), L_, H, W, _f32(out))
        return out, bool(bad)

    def footprints(self, cam, points):
        Pn = points.size // 3
        taps = np.zeros((Pn, 4), np.int32)
        valid = np.zeros(Pn, np.uint8)
        fr = np.zeros((Pn, 2), np.float64)
        c = _cams([cam])
        self.lib.lvso_footprints(c, _f32(points), Pn, taps.ctypes.data_as(vp),
                                 valid.ctypes.data_as(vp), fr.ctypes.data_as(vp))
        return taps, valid, fr

    def gather(self, cam, image, points):
        Hi, Wi, C = image.shape
        Pn = points.size // 3
        vals = np.zeros((Pn, C), np.float32)
        mask = np.zeros(Pn, np.float32)
        self.lib.lvso_gather(_cams([cam]), _f32(image), Hi, Wi, C, _f32(points), Pn, _f32(vals),
                             _f32(mask))
        return vals, mask

    def conv3x3(self, x, w, b):
        Cin, H, W = x.shape
        Cout = w.shape[0]
        y = np.zeros((Cout, H, W), np.float32)
        self.lib.lvso_conv3x3(_f32(x), _f32(w), _f32(b), _f32(y), Cin, Cout, H, W)
        return y

    def upsample_activate(self, fr, V, w_depth, w_sigma, logits, Ho, Wo):
        L_, H, W, C = V.shape
        M = logits.shape[-1]
        d = np.zeros((L_, Ho, Wo), np.float32)
        s = np.zeros((L_, Ho, Wo), np.float32)
        b = np.zeros((L_, Ho, Wo, M), np.float32)
        self.lib.lvso_upsample_activate(ctypes.byref(_fr(fr)), _f32(V), L_, H, W, C, _f32(w_depth),
                                        _f32(w_sigma), _f32(logits), M, Ho, Wo, _f32(d), _f32(s),
                                        _f32(b))
        return d, s, b

    def render_target(self, fr, depth, density, blend, images, cams):
        L_, Ho, Wo, M = blend.shape
        _, Hr, Wr, _ = images.shape
        rgb = np.zeros((Ho, Wo, 3), np.float32)
        bad = self.lib.lvso_render_target(ctypes.byref(_fr(fr)), _f32(depth), _f32(density),
                                          _f32(blend), L_, Ho, Wo, M, _f32(images), Hr, Wr,
                                          _cams(cams), _f32(rgb))
        return rgb, bool(bad)

    def trace_margins(self, tol, fn, cap=1 << 20):
        """Runs fn() with the validity-margin trace on (lvso_trace_margins):
        returns (fn's result, rows [n, 8] = step, kind (0 gather / 1 splat),
        view, layer, y, x, signed margin px, u-or-v)."""
        buf = np.zeros((cap, 8), np.float32)
        self.lib.lvso_trace_margins(float(tol), buf.ctypes.data_as(vp), cap)
        try:
            out = fn()
            n = int(self.lib.lvso_trace_count())
        finally:
            self.lib.lvso_trace_margins(0.0, None, 0)
        return out, buf[:min(n, cap)].copy()

    def attend_residual(self, V, deltas, wq, wo, gain, zero_scores=False):
        """V [P,C] (not modified) -> V + OTM(rms_norm(V)); deltas [P,M,C];
        wq [h,C,C]; wo [h*C,C]."""
        V = np.array(V, np.float32, copy=True, order="C")
        P_, C = V.shape
        M = deltas.shape[1]
        wq = np.ascontiguousarray(wq, np.float32)
        self.lib.lvso_attend_residual(_f32(V), _f32(np.ascontiguousarray(deltas)), P_, C, M,
                                      wq.shape[0], _f32(wq), _f32(np.ascontiguousarray(wo)),
                                      _f32(np.ascontiguousarray(gain)), int(zero_scores))
        return V

    def render_to_view(self, fr, V, w_appear, w_sigma, w_depth, cam):
        L_, H, W, C = V.shape
        Ca = w_appear.shape[1]
        out = np.zeros((cam.height, cam.width, Ca + 1), np.float32)
        bad = self.lib.lvso_render_to_view(ctypes.byref(_fr(fr)), _f32(V), L_, H, W, C, Ca,
                                           _f32(w_appear), _f32(w_sigma), _f32(w_depth),
                                           _cams([cam]), _f32(out))
        return out, bool(bad)


def _out_shapes(cfg, M, He, We):
    """Output extents of forward/render (network.cpp:118-150 restated)."""
    import math
    last = cfg.steps[-1]
    L_, H, W = last.layers, last.height, last.width
    Ho = int(math.floor(H * cfg.upsample + 0.5))
    Wo = int(math.floor(W * cfg.upsample + 0.5))
    C = cfg.channels
    return {"rgb": (Ho, Wo, 3), "depth": (L_, Ho, Wo), "density": (L_, Ho, Wo),
            "blend": (L_, Ho, Wo, M), "blend_logits": (L_, H, W, M), "volume": (L_, H, W, C),
            "deltas": (L_, H, W, M, C), "rgb_direct": (Ho, Wo, 3)}


def _forward_render(fn, cfg, enc_images, enc_cams, render_images, render_cams, target, weights,
                    outputs, errfirst):
    M, He, We, _ = enc_images.shape
    shapes = _out_shapes(cfg, M, He, We)
    outs = {k: np.zeros(shapes[k], np.float32) for k in outputs}
    cc = cfg.to_c()
    err = _Err()
    if render_images is not None:
        _, Hr, Wr, _ = render_images.shape
        rc = _cams(render_cams)
    else:
        Hr = Wr = 0
        rc = None
    args = [ctypes.byref(cc.c), M, _f32(enc_images), He, We, _cams(enc_cams), _f32(render_images),
            Hr, Wr, rc, ctypes.byref(_fr(target)), _f32(weights)]
    args += [_f32(outs.get(k)) for k in ("rgb", "depth", "density", "blend", "blend_logits",
                                          "volume", "deltas", "rgb_direct")]
    secs = (ctypes.c_double * 2)()
    if errfirst:
        args += [secs]
    args += [err.buf, 512]
    code = fn(*args)
    capi.raise_for(code, err.msg)
    if errfirst:
        outs["seconds"] = (secs[0], secs[1])
    return outs


class Reference:
    """The reference library itself (oracle/_ref/libref.so)."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (make -C oracle ref)")
        self.lib = ctypes.CDLL(REF_SO)
        L = self.lib
        cp, sz = ctypes.c_char_p, ctypes.c_size_t
        L.ref_param_count.argtypes = [P(capi.ModelConfigC), P(i64), P(i64), cp, sz]
        L.ref_init_param_store.argtypes = [P(capi.ModelConfigC), ctypes.c_uint64, vp, vp, vp, cp, sz]
        L.ref_plan_forward.argtypes = [P(capi.ModelConfigC), i64, i64, P(capi.PlanC), cp, sz]
        L.ref_rig.argtypes = [i64, i64, ctypes.c_double, i64, i64, ctypes.c_double, P(capi.CameraC),
                              P(capi.CameraC), cp, sz]
        L.ref_scene_images.argtypes = [ctypes.c_uint64, i64, P(capi.FrustumC), i64, P(capi.CameraC),
                                       vp, cp, sz]
        L.ref_scene_images_shifted.argtypes = [ctypes.c_uint64, i64, P(capi.FrustumC),
                                               ctypes.c_double, i64, P(capi.CameraC), vp, cp, sz]
        L.ref_attend_residual.argtypes = [vp, vp, i64, i64, i64, i64, vp, vp, vp, ctypes.c_int,
                                          cp, sz]
        L.ref_render_to_input_view.argtypes = [P(capi.FrustumC), vp, i64, i64, i64, i64, i64,
                                               vp, vp, vp, P(capi.CameraC), vp, cp, sz]
        L.ref_forward_render_ex.argtypes = [P(capi.ModelConfigC), i64, vp, i64, i64,
                                            P(capi.CameraC), vp, i64, i64, P(capi.CameraC),
                                            P(capi.FrustumC), vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                            vp, cp, sz]
        L.ref_model_config_to_json.argtypes = [P(capi.ModelConfigC), cp, sz, cp, sz]
        L.ref_model_config_roundtrip.argtypes = [cp, cp, sz, cp, sz]
        L.ref_pack_param_store.argtypes = [P(capi.ModelConfigC), ctypes.c_uint64, cp, vp, sz,
                                           P(sz), cp, sz]
        L.ref_qntc_roundtrip.argtypes = [cp, sz, vp, sz, P(sz), cp, sz]
        L.ref_resize_hwc.argtypes = [vp, i64, i64, i64, i64, i64, i64, vp, cp, sz]
        L.ref_world_points.argtypes = [P(capi.FrustumC), vp, i64, i64, i64, vp, cp, sz]
        L.ref_gather.argtypes = [P(capi.CameraC), vp, i64, i64, i64, vp, i64, vp, vp, cp, sz]
        L.ref_footprints.argtypes = [P(capi.CameraC), vp, i64, vp, vp, vp, cp, sz]
        L.ref_upsample_activate.argtypes = [P(capi.FrustumC), vp, i64, i64, i64, i64, vp, vp, vp,
                                            i64, i64, i64, vp, vp, vp, cp, sz]
        L.ref_render_target.argtypes = [P(capi.FrustumC), vp, vp, vp, i64, i64, i64, i64, vp, i64,
                                        i64, P(capi.CameraC), vp, cp, sz]

    def _call(self, fn, *args):
        err = _Err()
        code = fn(*args, err.buf, 512)
        capi.raise_for(code, err.msg)

    def init_param_store(self, cfg, seed):
        cc = cfg.to_c()
        n, tot = i64(), i64()
        self._call(self.lib.ref_param_count, ctypes.byref(cc.c), ctypes.byref(n), ctypes.byref(tot))
        out = np.zeros(tot.value, np.float32)
        ranks = np.zeros(n.value, np.int32)
        dims = np.zeros((n.value, 4), np.int64)
        self._call(self.lib.ref_init_param_store, ctypes.byref(cc.c), seed, _f32(out),
                   ranks.ctypes.data_as(vp), dims.ctypes.data_as(vp))
        return out, ranks, dims

    def model_config_to_json(self, cfg) -> str:
        cc = cfg.to_c()
        buf = ctypes.create_string_buffer(1 << 16)
        self._call(self.lib.ref_model_config_to_json, ctypes.byref(cc.c), buf, 1 << 16)
        return buf.value.decode()

    def pack_param_store(self, cfg, seed, names) -> bytes:
        """The reference's pack_tensors over its own init_param_store."""
        cc = cfg.to_c()
        n = sz()
        nm = "\n".join(names).encode()
        self._call(self.lib.ref_pack_param_store, ctypes.byref(cc.c), seed, nm, None, 0,
                   ctypes.byref(n))
        buf = ctypes.create_string_buffer(n.value)
        self._call(self.lib.ref_pack_param_store, ctypes.byref(cc.c), seed, nm, buf, n.value,
                   ctypes.byref(n))
        return buf.raw[:n.value]

    def resize_hwc(self, x, Ho, Wo):
        """The reference's resize_bilinear of [B,H,W,C] per channel."""
        x = np.ascontiguousarray(x, np.float32)
        B, H, W, C = x.shape
        out = np.zeros((B, Ho, Wo, C), np.float32)
        self._call(self.lib.ref_resize_hwc, _f32(x), B, H, W, C, Ho, Wo, _f32(out))
        return out

    def qntc_roundtrip(self, data: bytes) -> bytes:
        """pack_tensors(unpack_tensors(data)); raises the reference's
        IoError / SchemaError message (codes 3 / 1)."""
        n = sz()
        self._call(self.lib.ref_qntc_roundtrip, data, len(data), None, 0, ctypes.byref(n))
        buf = ctypes.create_string_buffer(max(n.value, 1))
        self._call(self.lib.ref_qntc_roundtrip, data, len(data), buf, n.value, ctypes.byref(n))
        return buf.raw[:n.value]

    def model_config_roundtrip(self, text: str) -> str:
        """model_config_to_json(model_config_from_json(text)); raises with the
        reference's SchemaError / DimError message on a rejected document."""
        buf = ctypes.create_string_buffer(1 << 16)
        self._call(self.lib.ref_model_config_roundtrip, text.encode(), buf, 1 << 16)
        return buf.value.decode()

    def plan_forward(self, cfg, h, w):
        cc = cfg.to_c()
        p = capi.PlanC()
        self._call(self.lib.ref_plan_forward, ctypes.byref(cc.c), h, w, ctypes.byref(p))
        return p

    def rig(self, rows, cols, baseline, width, height, focal):
        cams = (capi.CameraC * (rows * cols))()
        tgt = capi.CameraC()
        self._call(self.lib.ref_rig, rows, cols, baseline, width, height, focal, cams,
                   ctypes.byref(tgt))
        return list(cams), tgt

    def scene_images(self, seed, planes, scene_fr, cams, shift_x=0.0):
        M = len(cams)
        H, W = cams[0].height, cams[0].width
        out = np.zeros((M, H, W, 3), np.float32)
        self._call(self.lib.ref_scene_images_shifted, seed, planes, ctypes.byref(_fr(scene_fr)),
                   float(shift_x), M, _cams(cams), _f32(out))
        return out

    def forward_render(self, cfg, enc_images, enc_cams, render_images, render_cams, target,
                       weights, outputs=("rgb",)):
        def fn(*a):
            return self.lib.ref_forward_render_ex(*a)
        return _forward_render(fn, cfg, enc_images, enc_cams, render_images, render_cams, target,
                               weights, outputs, errfirst=True)

    def world_points(self, fr, depth):
        L_, H, W = depth.shape
        out = np.zeros((L_, H, W, 3), np.float32)
        self._call(self.lib.ref_world_points, ctypes.byref(_fr(fr)), _f32(depth), L_, H, W,
                   _f32(out))
        return out

    def footprints(self, cam, points):
        Pn = points.size // 3
        taps = np.zeros((Pn, 4), np.int32)
        valid = np.zeros(Pn, np.uint8)
        fr = np.zeros((Pn, 2), np.float64)
        self._call(self.lib.ref_footprints, _cams([cam]), _f32(points), Pn, taps.ctypes.data_as(vp),
                   valid.ctypes.data_as(vp), fr.ctypes.data_as(vp))
        return taps, valid, fr

    def gather(self, cam, image, points):
        Hi, Wi, C = image.shape
        Pn = points.size // 3
        vals = np.zeros((Pn, C), np.float32)
        mask = np.zeros(Pn, np.float32)
        self._call(self.lib.ref_gather, _cams([cam]), _f32(image), Hi, Wi, C, _f32(points), Pn,
                   _f32(vals), _f32(mask))
        return vals, mask

    def upsample_activate(self, fr, V, w_depth, w_sigma, logits, Ho, Wo):
        L_, H, W, C = V.shape
        M = logits.shape[-1]
        d = np.zeros((L_, Ho, Wo), np.float32)
        s = np.zeros((L_, Ho, Wo), np.float32)
        b = np.zeros((L_, Ho, Wo, M), np.float32)
        self._call(self.lib.ref_upsample_activate, ctypes.byref(_fr(fr)), _f32(V), L_, H, W, C,
                   _f32(w_depth), _f32(w_sigma), _f32(logits), M, Ho, Wo, _f32(d), _f32(s),
                   _f32(b))
        return d, s, b

    def render_target(self, fr, depth, density, blend, images, cams):
        L_, Ho, Wo, M = blend.shape
        _, Hr, Wr, _ = images.shape
        rgb = np.zeros((Ho, Wo, 3), np.float32)
        self._call(self.lib.ref_render_target, ctypes.byref(_fr(fr)), _f32(depth), _f32(density),
                   _f32(blend), L_, Ho, Wo, M, _f32(images), Hr, Wr, _cams(cams), _f32(rgb))
        return rgb

    def attend_residual(self, V, deltas, wq, wo, gain, zero_scores=False):
        V = np.array(V, np.float32, copy=True, order="C")
        P_, C = V.shape
        M = deltas.shape[1]
        wq = np.ascontiguousarray(wq, np.float32)
        self._call(self.lib.ref_attend_residual, _f32(V), _f32(np.ascontiguousarray(deltas)), P_,
                   C, M, wq.shape[0], _f32(wq), _f32(np.ascontiguousarray(wo)),
                   _f32(np.ascontiguousarray(gain)), int(zero_scores))
        return V

    def render_to_view(self, fr, V, w_appear, w_sigma, w_depth, cam):
        L_, H, W, C = V.shape
        Ca = w_appear.shape[1]
        out = np.zeros((cam.height, cam.width, Ca + 1), np.float32)
        self._call(self.lib.ref_render_to_input_view, ctypes.byref(_fr(fr)), _f32(V), L_, H, W,
                   C, Ca, _f32(w_appear), _f32(w_sigma), _f32(w_depth), _cams([cam]), _f32(out))
        return out


def fnv1a64(arr: np.ndarray) -> str:
    h = 14695981039346656037
    for b in arr.tobytes():
        h ^= b
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def fnv1a64_fast(arr: np.ndarray) -> str:
    """FNV-1a-64 over raw bytes, vectorised in chunks (same value as fnv1a64)."""
    data = np.frombuffer(arr.tobytes(), np.uint8)
    h = 14695981039346656037
    prime = 1099511628211
    mask = 0xFFFFFFFFFFFFFFFF
    for b in data.tolist():
        h = ((h ^ b) * prime) & mask
    return f"{h:016x}"
