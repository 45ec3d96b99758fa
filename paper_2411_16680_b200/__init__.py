"""B200-native drop-in for Quark's per-frame reconstruct + render path
(arXiv 2411.16680), behind the reference `lvs` library's API.

The compute lives in the in-tree native library liblvsg.so (hand-written
CUDA for sm_100a + C++ host runtime, C ABI in include/lvsg.h); this package
is its Python mirror. See DESIGN.md.
"""
from .camera import Camera, Frustum, RigSpec, pose_cam_from_world  # noqa: F401
from .capi import DeviceError, DimError, IoError, NumericError  # noqa: F401
from .config import (ModelConfig, SchemaError, StepConfig, config1,  # noqa: F401
                     full_scale_config, micro_config, model_config_from_json,
                     model_config_to_json, nano_config, scaled_full_config)
from .lvs import (Ldm, Model, init_param_store, param_shapes, plan_forward,  # noqa: F401
                  rig_cameras, scene_images, validate_config)
