"""Python mirror of the reference `lvs` C++ API for the per-frame path,
backed by the native library (liblvsg.so) through the C ABI of
include/lvsg.h.

  reference (proj/include/lvs)                 here
  ------------------------------------------  ----------------------------------
  plan_forward (network.cpp:105-151)           plan_forward(cfg, h, w)
  ModelConfig::validate (network.cpp:45-103)   validate_config(cfg)
  init_param_store (network.hpp:354-362)       init_param_store(cfg, seed)
  bind_params (network.hpp:330-339)            Model.load_weights(store)
  forward (network.hpp:562-603)                Model.forward(images, cams, target)
  render_target (ldm.hpp:193-199)              Model.render_target(images, cams)
  forward-demo (main.cpp:533-541)              Model.forward_render(...)
  RigSpec / make_scene / oracle_render         rig_cameras / scene_images

Errors map to the reference's classes: DimError (shape / contract),
NumericError, DeviceError. There is no CPU fallback: every compute call runs
the CUDA kernels of liblvsg.so on the context's GPU.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import capi
from .camera import Camera, Frustum, RigSpec
from .config import ModelConfig

vp = ctypes.c_void_p


def _err_buf():
    return ctypes.create_string_buffer(1024)


def validate_config(cfg: ModelConfig) -> None:
    cc = cfg.to_c()
    e = _err_buf()
    capi.raise_for(capi.lib().lvsg_validate_config(cc.ptr, e, 1024), e.value.decode())


@dataclass
class StepPlan:
    in_layers: int
    layers: int
    in_height: int
    in_width: int
    height: int
    width: int
    doubled: bool
    level: int
    feat_h: int
    feat_w: int
    render_h: int
    render_w: int
    collapse_count: int
    num_tokens: int


@dataclass
class ForwardPlan:
    pyramid: List[tuple]
    steps: List[StepPlan]
    out_height: int
    out_width: int


def plan_forward(cfg: ModelConfig, image_h: int, image_w: int) -> ForwardPlan:
    cc = cfg.to_c()
    p = capi.PlanC()
    e = _err_buf()
    capi.raise_for(capi.lib().lvsg_plan_forward(cc.ptr, image_h, image_w, ctypes.byref(p), e, 1024),
                   e.value.decode())
    steps = []
    for s in range(p.num_steps):
        sp = p.steps[s]
        steps.append(StepPlan(sp.in_layers, sp.layers, sp.in_height, sp.in_width, sp.height,
                              sp.width, bool(sp.doubled), sp.level, sp.feat_h, sp.feat_w,
                              sp.render_h, sp.render_w, sp.collapse_count, sp.num_tokens))
    pyr = [(p.pyramid_h[k], p.pyramid_w[k]) for k in range(p.num_levels)]
    return ForwardPlan(pyr, steps, p.out_height, p.out_width)


def param_shapes(cfg: ModelConfig) -> List[tuple]:
    cc = cfg.to_c()
    n, tot = ctypes.c_int64(), ctypes.c_int64()
    capi.raise_for(capi.lib().lvsg_param_count(cc.ptr, ctypes.byref(n), ctypes.byref(tot)),
                   "bad config")
    out = []
    rank = ctypes.c_int32()
    dims = (ctypes.c_int64 * 4)()
    for i in range(n.value):
        capi.lib().lvsg_param_shape(cc.ptr, i, ctypes.byref(rank), dims)
        out.append(tuple(dims[k] for k in range(rank.value)))
    return out


def init_param_store(cfg: ModelConfig, seed: int, flat: bool = False):
    """Bit-exact init_param_store<float>: a list of tensors in build_params
    order (or one flat array with flat=True)."""
    cc = cfg.to_c()
    n, tot = ctypes.c_int64(), ctypes.c_int64()
    capi.raise_for(capi.lib().lvsg_param_count(cc.ptr, ctypes.byref(n), ctypes.byref(tot)),
                   "bad config")
    buf = np.zeros(tot.value, np.float32)
    capi.raise_for(capi.lib().lvsg_init_param_store(cc.ptr, seed, buf.ctypes.data_as(capi.c_f32p)),
                   "bad config")
    if flat:
        return buf
    out, off = [], 0
    for shp in param_shapes(cfg):
        k = int(np.prod(shp))
        out.append(buf[off:off + k].reshape(shp))
        off += k
    return out


def rig_cameras(rig: RigSpec):
    """RigSpec::cameras() and ::target() (scenes.cpp:40-60)."""
    n = rig.rows * rig.cols
    cams = (capi.CameraC * n)()
    tgt = capi.CameraC()
    capi.raise_for(capi.lib().lvsg_rig_cameras(rig.rows, rig.cols, float(rig.baseline), rig.width,
                                               rig.height, float(rig.focal), cams,
                                               ctypes.byref(tgt)), "RigSpec")
    return [Camera.from_c(c) for c in cams], Camera.from_c(tgt)


def scene_images(seed: int, planes: int, scene_frustum: Frustum,
                 cams: Sequence[Camera], shift_x: float = 0.0) -> np.ndarray:
    """make_scene + oracle_render (scenes.cpp:62-171) -> [M, H, W, 3] f32.
    shift_x != 0 moves every plane but the backdrop wall along x (config 4's
    dynamic content)."""
    H, W = cams[0].height, cams[0].width
    assert all(c.height == H and c.width == W for c in cams)
    out = np.zeros((len(cams), H, W, 3), np.float32)
    arr = (capi.CameraC * len(cams))(*[c.to_c() for c in cams])
    e = _err_buf()
    L = capi.lib()
    fr = scene_frustum.to_c()
    capi.raise_for(L.lvsg_scene_images_shifted(seed, planes, ctypes.byref(fr), float(shift_x),
                                               len(cams), arr, out.ctypes.data_as(vp), e, 1024),
                   e.value.decode())
    return out


# cudaStreamLegacy: torch's default stream reports handle 0, which the C ABI
# reads as "the context's own stream"; pass the legacy default stream instead
# so the work really is ordered with the caller's stream (events, copies).
_CUDA_STREAM_LEGACY = 1


def _stream_handle(stream) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    h = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    return h if h else _CUDA_STREAM_LEGACY


def _cam_array(cams: Sequence[Camera]):
    return (capi.CameraC * len(cams))(*[c.to_c() for c in cams])


def _img_ptrs(images):
    """images: [M,H,W,3] array or a list of [H,W,3] arrays (host, f32)."""
    if isinstance(images, np.ndarray):
        if images.ndim != 4 or images.shape[-1] != 3:
            raise capi.DimError("images must be [M,H,W,3]")
        ims = [np.ascontiguousarray(images[m], np.float32) for m in range(images.shape[0])]
    else:
        ims = [np.ascontiguousarray(im, np.float32) for im in images]
    if not ims or any(im.ndim != 3 or im.shape[-1] != 3 for im in ims):
        raise capi.DimError("images must be [H,W,3]")
    H, W = ims[0].shape[:2]
    if any(im.shape[:2] != (H, W) for im in ims):
        raise capi.DimError("images must share one resolution")
    arr = (capi.c_f32p * len(ims))(*[im.ctypes.data_as(capi.c_f32p) for im in ims])
    return arr, ims, H, W


@dataclass
class Ldm:
    """Ldm<T> (ldm.hpp:14-21) plus the rest of ForwardResult
    (network.hpp:551-558): pre-softmax blend logits, final volume, the final
    step's deltas and, for direct_rgb configs, the decoded-colour composite
    `rgb` (None otherwise)."""
    depth: np.ndarray
    density: np.ndarray
    blend: np.ndarray
    blend_logits: np.ndarray
    volume: np.ndarray
    deltas: Optional[np.ndarray] = None
    rgb: Optional[np.ndarray] = None


class Model:
    """One lvsg context: device weights + stream + scratch arena for a
    ModelConfig (forward is single-caller per instance, as SPEC.md:531)."""

    def __init__(self, cfg: ModelConfig, device: int = 0):
        self.cfg = cfg
        self.device = int(device)
        self._cc = cfg.to_c()
        self._lib = capi.lib()
        h = ctypes.c_void_p()
        code = self._lib.lvsg_create(self._cc.ptr, int(device), ctypes.byref(h))
        capi.raise_for(code, (self._lib.lvsg_last_error(None) or b"").decode())
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            self._lib.lvsg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, code):
        if code != capi.OK:
            capi.raise_for(code, (self._lib.lvsg_last_error(self._h) or b"").decode())

    # --- weights (bind_params / init_params) ---
    def load_weights(self, store: Sequence[np.ndarray]) -> None:
        ts = [np.ascontiguousarray(t, np.float32) for t in store]
        ptrs = (capi.c_f32p * len(ts))(*[t.ctypes.data_as(capi.c_f32p) for t in ts])
        ranks = (ctypes.c_int32 * len(ts))(*[t.ndim for t in ts])
        dims_l = [d for t in ts for d in t.shape]
        dims = (ctypes.c_int64 * max(len(dims_l), 1))(*dims_l)
        self._check(self._lib.lvsg_load_weights(self._h, len(ts), ptrs, ranks, dims))

    def init_weights(self, seed: int) -> None:
        self._check(self._lib.lvsg_init_weights(self._h, seed))

    def load_weights_qntc(self, data: bytes) -> None:
        """A parameter store as a QNTC container (qntc.pack_tensors /
        the reference's pack_tensors), bound by position."""
        data = bytes(data)
        self._check(self._lib.lvsg_load_weights_qntc(self._h, data, len(data)))

    # --- forward / render ---
    def forward(self, images, cams: Sequence[Camera], target: Frustum,
                outputs: bool = True, deltas: bool = False) -> Optional[Ldm]:
        arr, keep, H, W = _img_ptrs(images)
        fr = target.to_c()
        out = None
        res = None
        if outputs:
            plan = plan_forward(self.cfg, H, W)
            last = plan.steps[-1]
            L_, Hh, Ww, M, C = last.layers, last.height, last.width, self.cfg.views, self.cfg.channels
            Ho, Wo = plan.out_height, plan.out_width
            res = Ldm(np.zeros((L_, Ho, Wo), np.float32), np.zeros((L_, Ho, Wo), np.float32),
                      np.zeros((L_, Ho, Wo, M), np.float32), np.zeros((L_, Hh, Ww, M), np.float32),
                      np.zeros((L_, Hh, Ww, C), np.float32),
                      np.zeros((L_, Hh, Ww, M, C), np.float32) if deltas else None,
                      np.zeros((Ho, Wo, 3), np.float32) if self.cfg.direct_rgb else None)
            out = capi.LdmOutC(*[a.ctypes.data_as(capi.c_f32p) if a is not None else None for a in
                                 (res.depth, res.density, res.blend, res.blend_logits, res.volume,
                                  res.deltas, res.rgb)])
        self._check(self._lib.lvsg_forward(self._h, len(keep), arr, H, W, _cam_array(cams),
                                           ctypes.byref(fr), ctypes.byref(out) if out else None))
        return res

    def render_target(self, images, cams: Sequence[Camera]) -> np.ndarray:
        arr, keep, H, W = _img_ptrs(images)
        plan_h, plan_w = self._out_hw()
        rgb = np.zeros((plan_h, plan_w, 3), np.float32)
        self._check(self._lib.lvsg_render(self._h, len(keep), arr, H, W, _cam_array(cams),
                                          rgb.ctypes.data_as(capi.c_f32p)))
        return rgb

    def forward_render(self, enc_images, enc_cams, render_images, render_cams,
                       target: Frustum, out: Optional[np.ndarray] = None,
                       enc_hw=None) -> np.ndarray:
        """Host buffers in, host RGB out (optionally into `out`, e.g. a view of
        pinned memory). enc_images=None: the resident pyramid of encode_device
        (complete on stream_handle()) at encoder resolution enc_hw."""
        if enc_images is None:
            ea, ek = None, [None] * self.cfg.views
            He, We = enc_hw
        else:
            ea, ek, He, We = _img_ptrs(enc_images)
        ra, rk, Hr, Wr = _img_ptrs(render_images)
        if out is None:
            plan = plan_forward(self.cfg, He, We)
            rgb = np.zeros((plan.out_height, plan.out_width, 3), np.float32)
        else:
            rgb = out
            assert rgb.dtype == np.float32 and rgb.flags.c_contiguous
        fr = target.to_c()
        self._last_enc_hw = (He, We)
        self._check(self._lib.lvsg_forward_render(self._h, len(ek), ea, He, We,
                                                  _cam_array(enc_cams), ra, Hr, Wr,
                                                  _cam_array(render_cams), ctypes.byref(fr),
                                                  rgb.ctypes.data_as(capi.c_f32p)))
        return rgb

    def forward_render_decimated(self, render_images, render_cams, target: Frustum,
                                 enc_hw, out: Optional[np.ndarray] = None) -> np.ndarray:
        """lvsg_forward_render_decimated: only the full-resolution views are
        passed; the encoder sees their resize_bilinear to enc_hw through
        Camera.scaled cameras."""
        ra, rk, Hr, Wr = _img_ptrs(render_images)
        He, We = enc_hw
        if out is None:
            plan = plan_forward(self.cfg, He, We)
            out = np.zeros((plan.out_height, plan.out_width, 3), np.float32)
        assert out.dtype == np.float32 and out.flags.c_contiguous
        fr = target.to_c()
        self._last_enc_hw = (He, We)
        self._check(self._lib.lvsg_forward_render_decimated(
            self._h, len(rk), ra, Hr, Wr, _cam_array(render_cams), He, We, ctypes.byref(fr),
            out.ctypes.data_as(capi.c_f32p)))
        return out

    def submit_frame_decimated(self, render_images, render_cams, target: Frustum, enc_hw,
                               out: np.ndarray) -> int:
        """lvsg_submit_frame_decimated: the pipelined form of
        forward_render_decimated; wait_frame(ticket) fills `out`."""
        ra, rk, Hr, Wr = _img_ptrs(render_images)
        assert out.dtype == np.float32 and out.flags.c_contiguous
        fr = target.to_c()
        t = ctypes.c_int64(-1)
        self._check(self._lib.lvsg_submit_frame_decimated(
            self._h, len(rk), ra, Hr, Wr, _cam_array(render_cams), enc_hw[0], enc_hw[1],
            ctypes.byref(fr), out.ctypes.data_as(capi.c_f32p), ctypes.byref(t)))
        self._inflight = getattr(self, "_inflight", {})
        self._inflight[t.value] = (ra, rk, out)
        return t.value

    def decimate_views_device(self, src, dst, stream=None) -> None:
        """lvsg_decimate_views_device on torch CUDA tensors [M,h,w,3] ->
        [M,out_h,out_w,3]."""
        for t in (src, dst):
            assert t.is_cuda and t.is_contiguous() and t.dtype.itemsize == 4 and t.shape[-1] == 3
        self._check(self._lib.lvsg_decimate_views_device(
            self._h, src.shape[0], src.data_ptr(), src.shape[1], src.shape[2], dst.data_ptr(),
            dst.shape[1], dst.shape[2], _stream_handle(stream)))

    def submit_frame(self, enc_images, enc_cams, render_images, render_cams, target: Frustum,
                     out: np.ndarray) -> int:
        """lvsg_submit_frame: enqueue one host-buffer frame (pinned arrays
        for overlap) and return its ticket; `out` [Ho,Wo,3] is filled by
        wait_frame(ticket). The arrays must stay alive until then."""
        ea, ek, He, We = _img_ptrs(enc_images)
        ra, rk, Hr, Wr = _img_ptrs(render_images)
        assert out.dtype == np.float32 and out.flags.c_contiguous
        fr = target.to_c()
        t = ctypes.c_int64(-1)
        self._check(self._lib.lvsg_submit_frame(self._h, len(ek), ea, He, We, _cam_array(enc_cams),
                                                ra, Hr, Wr, _cam_array(render_cams),
                                                ctypes.byref(fr), out.ctypes.data_as(capi.c_f32p),
                                                ctypes.byref(t)))
        self._inflight = getattr(self, "_inflight", {})
        self._inflight[t.value] = (ea, ek, ra, rk, out)  # keep the host views alive
        return t.value

    def wait_frame(self, ticket: int) -> None:
        try:
            self._check(self._lib.lvsg_wait_frame(self._h, int(ticket)))
        finally:
            getattr(self, "_inflight", {}).pop(int(ticket), None)

    def forward_render_device(self, enc_images, enc_cams, render_images, render_cams,
                              target: Frustum, rgb_out, stream=None, enc_hw=None,
                              rows=None) -> None:
        """Device-resident path on torch CUDA tensors (enc [M,He,We,3],
        render [M,Hr,Wr,3], rgb_out [Ho,Wo,3]); enqueued on `stream`
        (torch.cuda.Stream or raw handle; default: torch's current stream).
        enc_images=None: the resident pyramid of encode_device (encoder
        resolution enc_hw) is used instead of encoding. rows=(r0, r1): only
        those output rows are rendered, rgb_out [r1-r0, Wo, 3]
        (lvsg_forward_render_rows_device)."""
        import torch
        for t in (render_images, rgb_out) + ((enc_images,) if enc_images is not None else ()):
            if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
                raise capi.DimError("device tensors must be contiguous float32 CUDA tensors")
        sh = _stream_handle(stream)
        M, Hr, Wr, _ = render_images.shape
        if enc_images is not None:
            _, He, We, _ = enc_images.shape
            ep = enc_images.data_ptr()
        else:
            He, We = enc_hw
            ep = None
        fr = target.to_c()
        if rows is not None:
            self._check(self._lib.lvsg_forward_render_rows_device(
                self._h, M, ep, He, We, _cam_array(enc_cams),
                render_images.data_ptr(), Hr, Wr, _cam_array(render_cams), ctypes.byref(fr),
                int(rows[0]), int(rows[1]), rgb_out.data_ptr(), sh))
            return
        self._check(self._lib.lvsg_forward_render_device(
            self._h, M, ep, He, We, _cam_array(enc_cams),
            render_images.data_ptr(), Hr, Wr, _cam_array(render_cams), ctypes.byref(fr),
            rgb_out.data_ptr(), sh))

    def encode_device(self, enc_images, view0: int = 0, view1: Optional[int] = None,
                      stream=None) -> None:
        """encode_inputs' convolutions for views [view0, view1) of the device
        images [M,He,We,3] into the resident feature pyramid (lvsg_encode_device)."""
        M, He, We, _ = enc_images.shape
        self._check(self._lib.lvsg_encode_device(self._h, M, enc_images.data_ptr(), He, We, view0,
                                                 M if view1 is None else view1,
                                                 _stream_handle(stream)))

    def pyramid_export(self, enc_hw) -> bytes:
        """CUDA IPC handles of the pyramid level buffers (lvsg_pyramid_export):
        pyramid_levels x 64 bytes, to be handed to the other ranks."""
        n = self.cfg.pyramid_levels * 64
        buf = ctypes.create_string_buffer(n)
        self._check(self._lib.lvsg_pyramid_export(self._h, int(enc_hw[0]), int(enc_hw[1]), buf))
        return buf.raw[:n]

    def pyramid_import(self, peer_handles) -> None:
        """lvsg_pyramid_import: the other ranks' exported handles (a list of
        bytes); from then on encode_device writes its pooled levels into every
        peer's pyramid as well (the fused exchange)."""
        blob = b"".join(peer_handles) or None
        self._check(self._lib.lvsg_pyramid_import(self._h, len(peer_handles), blob))

    def pyramid_level(self, level: int):
        """Level `level` of the resident feature pyramid as a torch CUDA tensor
        [M, H_k, W_k, C] aliasing the context's buffer (e.g. for an NCCL
        all-gather of a view-sharded encode)."""
        import torch
        ptr = ctypes.c_void_p()
        dims = (ctypes.c_int64 * 4)()
        self._check(self._lib.lvsg_pyramid_level(self._h, level, ctypes.byref(ptr), dims))
        shape = tuple(int(d) for d in dims)

        class _Cai:  # __cuda_array_interface__ v3 view of the device buffer
            __cuda_array_interface__ = {"shape": shape, "typestr": "<f4", "data": (ptr.value, False),
                                        "version": 3, "strides": None, "stream": None}
        return torch.as_tensor(_Cai(), device=torch.device("cuda", self.device))

    def render_rows_device(self, render_images, render_cams, row0, row1, rgb_out, stream=None):
        sh = _stream_handle(stream)
        M, Hr, Wr, _ = render_images.shape
        self._check(self._lib.lvsg_render_rows_device(self._h, M, render_images.data_ptr(), Hr, Wr,
                                                      _cam_array(render_cams), row0, row1,
                                                      rgb_out.data_ptr(), sh))

    def stream_handle(self) -> int:
        """The context's own CUDA stream (cudaStream_t as int), e.g. for
        torch.cuda.ExternalStream."""
        return int(self._lib.lvsg_stream(self._h) or 0)

    def synchronize(self):
        self._check(self._lib.lvsg_synchronize(self._h))

    def profile(self, on: bool) -> None:
        self._check(self._lib.lvsg_profile_enable(self._h, 1 if on else 0))

    def profile_read(self) -> dict:
        """{stage: (device_ms, launches)} accumulated since the last read."""
        buf = ctypes.create_string_buffer(8192)
        self._check(self._lib.lvsg_profile_read(self._h, buf, 8192))
        out = {}
        for line in buf.value.decode().splitlines():
            k, ms, n = line.split()
            out[k] = (float(ms), int(n))
        return out

    def last_launch_count(self) -> int:
        return int(self._lib.lvsg_last_launch_count(self._h))

    def _out_hw(self):
        last = self.cfg.steps[-1]
        import math
        return (int(math.floor(last.height * self.cfg.upsample + 0.5)),
                int(math.floor(last.width * self.cfg.upsample + 0.5)))

    # --- per-stage entry points (device pointers) ---
    def stage_world_points(self, fr: Frustum, depth_t, points_t):
        L_, H, W = depth_t.shape
        f = fr.to_c()
        self._check(self._lib.lvsg_stage_world_points(self._h, ctypes.byref(f), depth_t.data_ptr(),
                                                      L_, H, W, points_t.data_ptr()))

    def stage_footprints(self, cam: Camera, points_t, taps_t, valid_t, fracs_t):
        c = cam.to_c()
        P = points_t.numel() // 3
        self._check(self._lib.lvsg_stage_footprints(self._h, ctypes.byref(c), points_t.data_ptr(), P,
                                                    taps_t.data_ptr(), valid_t.data_ptr(),
                                                    fracs_t.data_ptr()))

    def stage_conv3x3(self, x_t, w_t, b_t, y_t, impl: int = 0):
        """x [B,H,W,Cin] -> y [B,H,W,Cout] (device tensors); impl 0 auto,
        1 fp32 SIMT, 2 tcgen05 3xTF32."""
        B, H, W, Cin = x_t.shape
        Cout = w_t.shape[0]
        self._check(self._lib.lvsg_stage_conv3x3(self._h, x_t.data_ptr(), w_t.data_ptr(),
                                                 b_t.data_ptr() if b_t is not None else None,
                                                 y_t.data_ptr(), B, Cin, Cout, H, W, impl))

    def stage_conv3x3_fused(self, x_t, w_t, b_t, y_t, cin, ci0=0, norm_gain_t=None, gelu=False,
                            resid_t=None, impl: int = 0):
        """The solve's fused conv: x [B,H,W,pstride] (first `cin` channels),
        weight slice [:, ci0:ci0+cin] of w [Cout, w_cin, 3, 3], optional
        rms-norm input scale, GELU and residual (y = resid + conv)."""
        B, H, W, ps = x_t.shape
        Cout, w_cin = w_t.shape[0], w_t.shape[1]
        ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
        self._check(self._lib.lvsg_stage_conv3x3_fused(
            self._h, x_t.data_ptr(), ps, w_t.data_ptr(), w_cin, ci0, ptr(b_t), ptr(norm_gain_t),
            1 if gelu else 0, ptr(resid_t), y_t.data_ptr(), B, cin, Cout, H, W, impl))

    def stage_attend(self, V_t, deltas_t, wq_t, wo_t, gain_t, zero_scores=False):
        """attend_residual (attention.hpp:248-252) in place on V [P, C];
        deltas [P, M, C] in the reference layout; wq [h, C, C]; wo [h*C, C]."""
        P_, M = deltas_t.shape[0], deltas_t.shape[1]
        self._check(self._lib.lvsg_stage_attend(self._h, V_t.data_ptr(), deltas_t.data_ptr(), P_,
                                                M, wq_t.shape[0], wq_t.data_ptr(),
                                                wo_t.data_ptr(), gain_t.data_ptr(),
                                                1 if zero_scores else 0))

    def stage_upsample_render(self, target: Frustum, V_t, logits_t, w_depth_t, w_sigma_t,
                              images_t, cams: Sequence[Camera], rgb_t):
        """upsample_activate + render_target (ldm.hpp:193-199, :249-271) of
        the final volume V [L,H,W,C] and logits [L,H,W,M] into rgb [Ho,Wo,3]."""
        L_, H, W, _ = V_t.shape
        M = logits_t.shape[-1]
        _, Hr, Wr, _ = images_t.shape
        Ho, Wo, _ = rgb_t.shape
        f = target.to_c()
        self._check(self._lib.lvsg_stage_upsample_render(
            self._h, ctypes.byref(f), V_t.data_ptr(), logits_t.data_ptr(), L_, H, W, M,
            w_depth_t.data_ptr(), w_sigma_t.data_ptr(), images_t.data_ptr(), Hr, Wr,
            _cam_array(cams), Ho, Wo, rgb_t.data_ptr()))

    def stage_render_to_view(self, target: Frustum, V_t, w_appear_t, w_sigma_t, w_depth_t,
                             cam: Camera, out_t):
        """render_to_input_view (ldm.hpp:223-244) of V [L,H,W,C] into one
        camera: out [cam.height, cam.width, Ca+1]."""
        L_, H, W, _ = V_t.shape
        f, c = target.to_c(), cam.to_c()
        self._check(self._lib.lvsg_stage_render_to_view(
            self._h, ctypes.byref(f), V_t.data_ptr(), L_, H, W, w_appear_t.data_ptr(),
            w_appear_t.shape[1], w_sigma_t.data_ptr(), w_depth_t.data_ptr(), ctypes.byref(c),
            out_t.data_ptr()))

    def stage_gather(self, cam: Camera, image_t, points_t, values_t, mask_t):
        c = cam.to_c()
        Hi, Wi, C = image_t.shape
        P = points_t.numel() // 3
        self._check(self._lib.lvsg_stage_gather(self._h, ctypes.byref(c), image_t.data_ptr(), Hi, Wi,
                                                C, points_t.data_ptr(), P, values_t.data_ptr(),
                                                mask_t.data_ptr()))
