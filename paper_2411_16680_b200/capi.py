"""ctypes mirror of include/lvsg.h and the loader for the in-tree native
library (paper_2411_16680_b200/liblvsg.so).

The product path has no CPU fallback: if the library is missing, `lib()`
raises. The struct layouts below must match include/lvsg.h exactly.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# LVSG_LIB overrides the library path (development probes of alternative builds).
LIB_PATH = os.environ.get("LVSG_LIB") or os.path.join(_HERE, "liblvsg.so")

c_i64 = ctypes.c_int64
c_i32 = ctypes.c_int32
c_f64 = ctypes.c_double
c_f32p = ctypes.POINTER(ctypes.c_float)


class StepConfig(ctypes.Structure):
    _fields_ = [("in_layers", c_i64), ("layers", c_i64), ("height", c_i64), ("width", c_i64),
                ("pyramid_level", c_i64), ("blocks", ctypes.c_char_p)]


class ModelConfigC(ctypes.Structure):
    _fields_ = [("steps", ctypes.POINTER(StepConfig)), ("num_steps", c_i64),
                ("channels", c_i64), ("views", c_i64), ("pyramid_levels", c_i64),
                ("upsample", c_f64), ("near_depth", c_f64), ("far_depth", c_f64),
                ("ablate_render", c_i32), ("ablate_attention", c_i32), ("ablate_rays", c_i32),
                ("direct_rgb", c_i32)]


class CameraC(ctypes.Structure):
    _fields_ = [("fx", c_f64), ("fy", c_f64), ("cx", c_f64), ("cy", c_f64), ("width", c_i64),
                ("height", c_i64), ("cam_from_world", c_f64 * 16)]


class FrustumC(ctypes.Structure):
    _fields_ = [("camera", CameraC), ("near_depth", c_f64), ("far_depth", c_f64)]


class StepPlanC(ctypes.Structure):
    _fields_ = [("in_layers", c_i64), ("layers", c_i64), ("in_height", c_i64),
                ("in_width", c_i64), ("height", c_i64), ("width", c_i64), ("doubled", c_i32),
                ("level", c_i64), ("feat_h", c_i64), ("feat_w", c_i64), ("render_h", c_i64),
                ("render_w", c_i64), ("collapse_count", c_i64), ("num_tokens", c_i64)]


MAX_STEPS = 32
MAX_LEVELS = 16


class PlanC(ctypes.Structure):
    _fields_ = [("num_levels", c_i64), ("pyramid_h", c_i64 * MAX_LEVELS),
                ("pyramid_w", c_i64 * MAX_LEVELS), ("num_steps", c_i64),
                ("steps", StepPlanC * MAX_STEPS), ("out_height", c_i64), ("out_width", c_i64)]


class LdmOutC(ctypes.Structure):
    _fields_ = [("depth", c_f32p), ("density", c_f32p), ("blend", c_f32p),
                ("blend_logits", c_f32p), ("volume", c_f32p), ("deltas", c_f32p),
                ("rgb", c_f32p)]


# Error classes (include/lvsg.h; reference tensor.hpp:15-25).
OK, ERR_DIM, ERR_NUMERIC, ERR_IO = 0, 1, 2, 3
ERR_CUDA, ERR_NO_DEVICE, ERR_NCCL, ERR_INTERNAL = 10, 11, 12, 13


class DimError(ValueError):
    """Shape / contract violation (reference DimError, tensor.hpp:15-19)."""


class NumericError(ArithmeticError):
    """NaN / Inf (reference NumericError, tensor.hpp:21-25)."""


class IoError(OSError):
    """Corrupt / truncated container (reference IoError, io.hpp:20-24)."""


class DeviceError(RuntimeError):
    """CUDA / NCCL / runtime failure in the native library."""


def raise_for(code: int, msg: str):
    if code == OK:
        return
    if code == ERR_DIM:
        raise DimError(msg)
    if code == ERR_NUMERIC:
        raise NumericError(msg)
    if code == ERR_IO:
        raise IoError(msg)
    raise DeviceError(f"lvsg error {code}: {msg}")


_lib = None

# Exported symbols of include/lvsg.h (checked by tests/test_capi.py).
SYMBOLS = [
    "lvsg_validate_config", "lvsg_plan_forward", "lvsg_param_count", "lvsg_param_shape",
    "lvsg_init_param_store", "lvsg_create", "lvsg_destroy", "lvsg_last_error",
    "lvsg_load_weights", "lvsg_init_weights", "lvsg_forward", "lvsg_render",
    "lvsg_forward_render", "lvsg_forward_render_device", "lvsg_render_rows_device",
    "lvsg_encode_device", "lvsg_pyramid_level", "lvsg_submit_frame", "lvsg_wait_frame",
    "lvsg_pyramid_export", "lvsg_pyramid_import",
    "lvsg_synchronize", "lvsg_last_launch_count", "lvsg_stream", "lvsg_stage_world_points",
    "lvsg_stage_footprints", "lvsg_stage_gather", "lvsg_rig_cameras", "lvsg_scene_images",
    "lvsg_scene_images_shifted", "lvsg_stage_attend", "lvsg_stage_upsample_render",
    "lvsg_stage_render_to_view", "lvsg_forward_render_rows_device",
    "lvsg_profile_enable", "lvsg_profile_read", "lvsg_stage_conv3x3", "lvsg_stage_conv3x3_fused",
    "lvsg_load_weights_qntc", "lvsg_param_name", "lvsg_pack_param_store_qntc",
    "lvsg_forward_render_decimated", "lvsg_submit_frame_decimated", "lvsg_decimate_views_device",
]


def lib() -> ctypes.CDLL:
    """Loads liblvsg.so (built in-tree by __graft_entry__.build()). Raises if
    it is missing: there is no fallback implementation."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; "
                          f"g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    vp = ctypes.c_void_p
    L.lvsg_validate_config.argtypes = [P(ModelConfigC), ctypes.c_char_p, ctypes.c_size_t]
    L.lvsg_plan_forward.argtypes = [P(ModelConfigC), c_i64, c_i64, P(PlanC), ctypes.c_char_p,
                                    ctypes.c_size_t]
    L.lvsg_param_count.argtypes = [P(ModelConfigC), P(c_i64), P(c_i64)]
    L.lvsg_param_shape.argtypes = [P(ModelConfigC), c_i64, P(c_i32), P(c_i64)]
    L.lvsg_init_param_store.argtypes = [P(ModelConfigC), ctypes.c_uint64, c_f32p]
    L.lvsg_create.argtypes = [P(ModelConfigC), c_i32, P(vp)]
    L.lvsg_destroy.argtypes = [vp]
    L.lvsg_destroy.restype = None
    L.lvsg_last_error.argtypes = [vp]
    L.lvsg_last_error.restype = ctypes.c_char_p
    L.lvsg_load_weights.argtypes = [vp, c_i64, P(c_f32p), P(c_i32), P(c_i64)]
    L.lvsg_init_weights.argtypes = [vp, ctypes.c_uint64]
    L.lvsg_load_weights_qntc.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t]
    L.lvsg_param_name.argtypes = [P(ModelConfigC), c_i64, ctypes.c_char_p, ctypes.c_size_t]
    L.lvsg_pack_param_store_qntc.argtypes = [P(ModelConfigC), ctypes.c_uint64, vp, ctypes.c_size_t,
                                             P(ctypes.c_size_t)]
    L.lvsg_forward.argtypes = [vp, c_i64, P(c_f32p), c_i64, c_i64, P(CameraC), P(FrustumC),
                               P(LdmOutC)]
    L.lvsg_render.argtypes = [vp, c_i64, P(c_f32p), c_i64, c_i64, P(CameraC), c_f32p]
    L.lvsg_forward_render.argtypes = [vp, c_i64, P(c_f32p), c_i64, c_i64, P(CameraC), P(c_f32p),
                                      c_i64, c_i64, P(CameraC), P(FrustumC), c_f32p]
    L.lvsg_forward_render_device.argtypes = [vp, c_i64, vp, c_i64, c_i64, P(CameraC), vp, c_i64,
                                             c_i64, P(CameraC), P(FrustumC), vp, vp]
    L.lvsg_render_rows_device.argtypes = [vp, c_i64, vp, c_i64, c_i64, P(CameraC), c_i64, c_i64,
                                          vp, vp]
    L.lvsg_forward_render_rows_device.argtypes = [vp, c_i64, vp, c_i64, c_i64, P(CameraC), vp,
                                                  c_i64, c_i64, P(CameraC), P(FrustumC), c_i64,
                                                  c_i64, vp, vp]
    L.lvsg_submit_frame.argtypes = [vp, c_i64, P(c_f32p), c_i64, c_i64, P(CameraC), P(c_f32p),
                                    c_i64, c_i64, P(CameraC), P(FrustumC), c_f32p, P(c_i64)]
    L.lvsg_wait_frame.argtypes = [vp, c_i64]
    L.lvsg_forward_render_decimated.argtypes = [vp, c_i64, P(c_f32p), c_i64, c_i64, P(CameraC),
                                                c_i64, c_i64, P(FrustumC), c_f32p]
    L.lvsg_submit_frame_decimated.argtypes = [vp, c_i64, P(c_f32p), c_i64, c_i64, P(CameraC),
                                              c_i64, c_i64, P(FrustumC), c_f32p, P(c_i64)]
    L.lvsg_decimate_views_device.argtypes = [vp, c_i64, vp, c_i64, c_i64, vp, c_i64, c_i64, vp]
    L.lvsg_encode_device.argtypes = [vp, c_i64, vp, c_i64, c_i64, c_i64, c_i64, vp]
    L.lvsg_pyramid_level.argtypes = [vp, c_i64, P(vp), P(c_i64)]
    L.lvsg_pyramid_export.argtypes = [vp, c_i64, c_i64, ctypes.c_char_p]
    L.lvsg_pyramid_import.argtypes = [vp, c_i64, ctypes.c_char_p]
    L.lvsg_synchronize.argtypes = [vp]
    L.lvsg_last_launch_count.argtypes = [vp]
    L.lvsg_last_launch_count.restype = c_i64
    L.lvsg_stream.argtypes = [vp]
    L.lvsg_stream.restype = vp
    L.lvsg_stage_world_points.argtypes = [vp, P(FrustumC), vp, c_i64, c_i64, c_i64, vp]
    L.lvsg_stage_footprints.argtypes = [vp, P(CameraC), vp, c_i64, vp, vp, vp]
    L.lvsg_stage_gather.argtypes = [vp, P(CameraC), vp, c_i64, c_i64, c_i64, vp, c_i64, vp, vp]
    L.lvsg_rig_cameras.argtypes = [c_i64, c_i64, c_f64, c_i64, c_i64, c_f64, P(CameraC),
                                   P(CameraC)]
    L.lvsg_scene_images.argtypes = [ctypes.c_uint64, c_i64, P(FrustumC), c_i64, P(CameraC), vp,
                                    ctypes.c_char_p, ctypes.c_size_t]
    L.lvsg_scene_images_shifted.argtypes = [ctypes.c_uint64, c_i64, P(FrustumC), c_f64, c_i64,
                                            P(CameraC), vp, ctypes.c_char_p, ctypes.c_size_t]
    L.lvsg_stage_attend.argtypes = [vp, vp, vp, c_i64, c_i64, c_i64, vp, vp, vp, c_i32]
    L.lvsg_stage_upsample_render.argtypes = [vp, P(FrustumC), vp, vp, c_i64, c_i64, c_i64, c_i64,
                                             vp, vp, vp, c_i64, c_i64, P(CameraC), c_i64, c_i64,
                                             vp]
    L.lvsg_stage_render_to_view.argtypes = [vp, P(FrustumC), vp, c_i64, c_i64, c_i64, vp, c_i64,
                                            vp, vp, P(CameraC), vp]
    L.lvsg_profile_enable.argtypes = [vp, c_i32]
    L.lvsg_profile_read.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t]
    L.lvsg_stage_conv3x3.argtypes = [vp, vp, vp, vp, vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_i32]
    L.lvsg_stage_conv3x3_fused.argtypes = [vp, vp, c_i64, vp, c_i64, c_i64, vp, vp, c_i32, vp, vp,
                                           c_i64, c_i64, c_i64, c_i64, c_i64, c_i32]
    _lib = L
    return L
