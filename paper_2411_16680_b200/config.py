"""ModelConfig / StepConfig mirror of the reference (network.hpp:38-59) and the
presets the benchmarks and tests run on.

The validation and planning rules themselves live in the native host library
(csrc/host.cpp: `lvsg_validate_config`, `lvsg_plan_forward`, restating
network.cpp:8-151); this module only carries the values across the C ABI.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field, replace
from typing import List

from . import capi


@dataclass
class StepConfig:
    """network.hpp:38-44."""

    in_layers: int
    layers: int
    height: int
    width: int
    pyramid_level: int
    blocks: str


@dataclass
class ModelConfig:
    """network.hpp:46-59 (`near`/`far` keep the reference names)."""

    steps: List[StepConfig] = field(default_factory=list)
    channels: int = 0
    views: int = 0
    pyramid_levels: int = 0
    upsample: float = 1.0
    near: float = 0.0
    far: float = 0.0
    ablate_render: bool = False
    ablate_attention: bool = False
    ablate_rays: bool = False
    direct_rgb: bool = False

    def with_views(self, m: int) -> "ModelConfig":
        return replace(self, views=m, steps=list(self.steps))

    # --- C ABI ---------------------------------------------------------------
    def to_c(self) -> "CConfig":
        return CConfig(self)


class CConfig:
    """Owns the ctypes storage behind an lvsg_model_config."""

    def __init__(self, cfg: ModelConfig):
        n = len(cfg.steps)
        self._blocks = [s.blocks.encode() for s in cfg.steps]
        self._steps = (capi.StepConfig * max(n, 1))()
        for i, s in enumerate(cfg.steps):
            self._steps[i] = capi.StepConfig(s.in_layers, s.layers, s.height, s.width,
                                             s.pyramid_level, self._blocks[i])
        self.c = capi.ModelConfigC(
            ctypes.cast(self._steps, ctypes.POINTER(capi.StepConfig)), n, cfg.channels,
            cfg.views, cfg.pyramid_levels, float(cfg.upsample), float(cfg.near), float(cfg.far),
            int(cfg.ablate_render), int(cfg.ablate_attention), int(cfg.ablate_rays),
            int(cfg.direct_rgb))

    @property
    def ptr(self):
        return ctypes.byref(self.c)


def nano_config() -> ModelConfig:
    """network.cpp:153-168."""
    return ModelConfig(
        steps=[StepConfig(8, 8, 8, 8, 2, "Bp,A2,C"),
               StepConfig(8, 8, 8, 8, 2, "U,A2,C,C"),
               StepConfig(8, 8, 16, 16, 1, "U,A2,C"),
               StepConfig(8, 4, 32, 32, 0, "Lc,U,A1,C")],
        channels=8, views=4, pyramid_levels=3, upsample=2.0, near=1.0, far=6.0)


def full_scale_config() -> ModelConfig:
    """network.cpp:170-187 (Table 6 schedule, 1080p output from 576x960 input)."""
    return ModelConfig(
        steps=[StepConfig(24, 24, 36, 64, 3, "Bp,A4,C,C,A4,C,C,A4,C,C"),
               StepConfig(24, 24, 36, 64, 3, "U,A4,C,C,A4,C,C,A4,C,C"),
               StepConfig(24, 24, 72, 128, 2, "U,A4,C,C,A4,C,C,A4,C,C"),
               StepConfig(24, 24, 72, 128, 2, "U,A4,C,A4,C"),
               StepConfig(24, 12, 144, 256, 1, "Lc,U,A2,C,A2,C"),
               StepConfig(12, 6, 288, 512, 0, "Lc,U,A1,C,A1,C")],
        channels=32, views=8, pyramid_levels=4, upsample=3.75, near=0.5, far=100.0)


def config1() -> ModelConfig:
    """BASELINE config 1: 4 views 256^2, C=32, Bp + 2 U&F steps."""
    return ModelConfig(
        steps=[StepConfig(8, 8, 32, 32, 2, "Bp,A4,C,C"),
               StepConfig(8, 8, 64, 64, 1, "U,A2,C"),
               StepConfig(8, 4, 64, 64, 1, "Lc,U,A1,C")],
        channels=32, views=4, pyramid_levels=3, upsample=4.0, near=1.0, far=20.0)


def micro_config() -> ModelConfig:
    """tests/test_network.cpp:27-40 (2 views, C=4)."""
    return ModelConfig(
        steps=[StepConfig(2, 2, 4, 4, 1, "Bp,A1,C"), StepConfig(2, 2, 8, 8, 0, "U,A1,C")],
        channels=4, views=2, pyramid_levels=2, upsample=1.0, near=1.0, far=5.0)


def scaled_full_config(div: int = 4) -> ModelConfig:
    """full_scale_config with every volume extent divided by `div` (same
    schedule, layers, channels and views; 1/div^2 of the texels). Used as the
    bounded CPU-baseline sample of config 2 (encoder input 576/div x 960/div)."""
    base = full_scale_config()
    steps = [StepConfig(s.in_layers, s.layers, s.height // div, s.width // div, s.pyramid_level,
                        s.blocks) for s in base.steps]
    return replace(base, steps=steps)


# --- ModelConfig JSON (io.cpp:571-633) ----------------------------------------

class SchemaError(ValueError):
    """A config document that does not fit the schema (reference SchemaError,
    io.hpp:28-31): bad JSON, a missing / mistyped / unknown field, or a
    config that fails ModelConfig::validate ("$: ..." prefix)."""


class _ObjView:
    """io.cpp:345-402: typed field access that records what it consumed, so
    close() can reject stray fields by name."""

    def __init__(self, j, path):
        if not isinstance(j, dict):
            raise SchemaError(f"{path}: expected an object")
        self.j, self.path, self.seen = j, path, set()

    def _get(self, key):
        self.seen.add(key)
        if key not in self.j:
            raise SchemaError(f"{self.path}.{key}: missing field")
        return self.j[key]

    def num(self, key):
        v = self._get(key)
        if isinstance(v, bool) or not isinstance(v, (int, float)):
            raise SchemaError(f"{self.path}.{key}: expected a number")
        return float(v)

    def integer(self, key):
        v = self._get(key)
        if isinstance(v, bool) or not isinstance(v, int):
            raise SchemaError(f"{self.path}.{key}: expected an integer")
        return int(v)

    def boolean(self, key, fallback):
        self.seen.add(key)
        if key not in self.j:
            return fallback
        v = self.j[key]
        if not isinstance(v, bool):
            raise SchemaError(f"{self.path}.{key}: expected a boolean")
        return v

    def str(self, key):
        v = self._get(key)
        if not isinstance(v, str):
            raise SchemaError(f"{self.path}.{key}: expected a string")
        return v

    def array(self, key, min_len=0):
        v = self._get(key)
        if not isinstance(v, list):
            raise SchemaError(f"{self.path}.{key}: expected an array")
        if len(v) < min_len:
            raise SchemaError(f"{self.path}.{key}: expected at least {min_len} entries")
        return v

    def close(self):
        for k in self.j:
            if k not in self.seen:
                raise SchemaError(f'{self.path}: unknown field "{k}"')


def model_config_to_json(cfg: ModelConfig) -> str:
    """model_config_to_json (io.cpp:571-596): the same fields, 2-space indent,
    keys in nlohmann's (sorted) order, trailing newline."""
    import json
    d = {"channels": cfg.channels, "views": cfg.views, "pyramid_levels": cfg.pyramid_levels,
         "upsample": float(cfg.upsample), "near": float(cfg.near), "far": float(cfg.far),
         "ablate_render": cfg.ablate_render, "ablate_attention": cfg.ablate_attention,
         "ablate_rays": cfg.ablate_rays, "direct_rgb": cfg.direct_rgb,
         "steps": [{"in_layers": s.in_layers, "layers": s.layers, "height": s.height,
                    "width": s.width, "pyramid_level": s.pyramid_level, "blocks": s.blocks}
                   for s in cfg.steps]}
    return json.dumps(d, indent=2, sort_keys=True) + "\n"


def model_config_from_json(text: str) -> ModelConfig:
    """model_config_from_json (io.cpp:598-633): schema-checked parse, then
    ModelConfig::validate through the native library (DimError -> SchemaError)."""
    import json
    try:
        j = json.loads(text)
    except ValueError as e:
        raise SchemaError(f"invalid json: {e}") from None
    ov = _ObjView(j, "$")
    cfg = ModelConfig(channels=ov.integer("channels"), views=ov.integer("views"),
                      pyramid_levels=ov.integer("pyramid_levels"), upsample=ov.num("upsample"),
                      near=ov.num("near"), far=ov.num("far"),
                      ablate_render=ov.boolean("ablate_render", False),
                      ablate_attention=ov.boolean("ablate_attention", False),
                      ablate_rays=ov.boolean("ablate_rays", False),
                      direct_rgb=ov.boolean("direct_rgb", False))
    steps = ov.array("steps", 1)
    for i, sj in enumerate(steps):
        sv = _ObjView(sj, f"$.steps[{i}]")
        cfg.steps.append(StepConfig(sv.integer("in_layers"), sv.integer("layers"),
                                    sv.integer("height"), sv.integer("width"),
                                    sv.integer("pyramid_level"), sv.str("blocks")))
        sv.close()
    ov.close()
    from .lvs import validate_config
    try:
        validate_config(cfg)
    except capi.DimError as e:
        raise SchemaError(f"$: {e}") from None
    return cfg
