"""Camera / Frustum value types mirroring camera.hpp:14-59 (pinhole, z-depth,
texel centres at +0.5, row-major cam_from_world), plus the synthetic camera
rigs the benchmarks use (RigSpec, scenes.hpp:46-60)."""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import capi


@dataclass
class Camera:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    cam_from_world: np.ndarray = field(default_factory=lambda: np.eye(4))

    @staticmethod
    def make(fx, fy, cx, cy, width, height, cam_from_world=None) -> "Camera":
        c = Camera(float(fx), float(fy), float(cx), float(cy), int(width), int(height),
                   np.eye(4) if cam_from_world is None else np.asarray(cam_from_world, np.float64))
        c.validate()
        return c

    def validate(self) -> None:
        """camera.cpp:19-29."""
        if self.fx <= 0 or self.fy <= 0:
            raise capi.DimError("camera: focal lengths must be positive")
        if self.width <= 0 or self.height <= 0:
            raise capi.DimError("camera: image size must be positive")
        R = self.cam_from_world[:3, :3]
        if np.abs(R.T @ R - np.eye(3)).max() >= 1e-5:
            raise capi.DimError("camera: rotation block not orthonormal")
        if np.abs(self.cam_from_world[3] - np.array([0, 0, 0, 1.0])).max() > 1e-12:
            raise capi.DimError("camera: transform bottom row must be (0,0,0,1)")

    def scaled(self, new_width: int, new_height: int) -> "Camera":
        """camera.cpp:67-78 (anisotropic re-digitisation)."""
        sx = float(new_width) / float(self.width)
        sy = float(new_height) / float(self.height)
        return Camera(self.fx * sx, self.fy * sy, self.cx * sx, self.cy * sy, int(new_width),
                      int(new_height), self.cam_from_world.copy())

    def to_c(self) -> capi.CameraC:
        c = capi.CameraC()
        c.fx, c.fy, c.cx, c.cy = self.fx, self.fy, self.cx, self.cy
        c.width, c.height = self.width, self.height
        flat = np.ascontiguousarray(self.cam_from_world, np.float64).reshape(-1)
        for i in range(16):
            c.cam_from_world[i] = float(flat[i])
        return c

    @staticmethod
    def from_c(c: capi.CameraC) -> "Camera":
        return Camera(c.fx, c.fy, c.cx, c.cy, c.width, c.height,
                      np.array(list(c.cam_from_world), np.float64).reshape(4, 4))


def pose_cam_from_world(world_R_cam: np.ndarray, center) -> np.ndarray:
    """camera.hpp:44-50."""
    m = np.eye(4)
    Rt = np.asarray(world_R_cam, np.float64).T
    m[:3, :3] = Rt
    c = np.asarray(center, np.float64)
    # k-ascending product of (-R^T) and c, as the oracle build computes it
    for r in range(3):
        acc = (-Rt[r, 0]) * c[0]
        acc += (-Rt[r, 1]) * c[1]
        acc += (-Rt[r, 2]) * c[2]
        m[r, 3] = acc
    return m


@dataclass
class Frustum:
    camera: Camera
    near: float
    far: float

    def validate(self) -> None:
        """camera.cpp:80-83."""
        self.camera.validate()
        if not (self.near > 0 and self.far > self.near):
            raise capi.DimError("frustum: requires 0 < near < far")

    def to_c(self) -> capi.FrustumC:
        f = capi.FrustumC()
        f.camera = self.camera.to_c()
        f.near_depth, f.far_depth = float(self.near), float(self.far)
        return f


@dataclass
class RigSpec:
    """scenes.hpp:46-60 / scenes.cpp:40-60: planar grid at z=0 facing +z."""

    rows: int = 1
    cols: int = 2
    baseline: float = 0.1
    width: int = 64
    height: int = 64
    focal: float = 64.0

    def cameras(self):
        cams = []
        for r in range(self.rows):
            for c in range(self.cols):
                x = (float(c) - float(self.cols - 1) / 2.0) * self.baseline
                y = (float(r) - float(self.rows - 1) / 2.0) * self.baseline
                cams.append(Camera.make(self.focal, self.focal, self.width / 2.0, self.height / 2.0,
                                        self.width, self.height,
                                        pose_cam_from_world(np.eye(3), (x, y, 0.0))))
        return cams

    def target(self) -> Camera:
        return Camera.make(self.focal, self.focal, self.width / 2.0, self.height / 2.0, self.width,
                           self.height, np.eye(4))
