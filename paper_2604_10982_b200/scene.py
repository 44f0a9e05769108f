"""Synthetic workloads: make_street_scene (proj/src/synthetic.cpp:236-312) and the
closed-form C5 camera trajectory. Host-only (no GPU needed)."""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np

from . import _abi as A
from . import _lib
from .raster import Camera, SceneMap, _check


@dataclass
class StreetSpec:  # synthetic.hpp:49-56 (+ scale_mult)
    n_surfels: int = 12000
    seed: int = 7
    min_aspect: float = 5.0
    image_w: int = 256
    image_h: int = 192
    c_sem: int = 32
    n_instances: int = 256
    scale_mult: float = 1.0

    def to_c(self) -> A.psm_street_spec:
        return A.psm_street_spec(int(self.n_surfels), int(self.seed), float(self.min_aspect), int(self.image_w),
                                 int(self.image_h), int(self.c_sem), int(self.n_instances), float(self.scale_mult))


def density_scale(n_surfels: int, width: int, height: int) -> float:
    """k(N, W, H) = sqrt((12000/N) * (256 H) / (192 W)): keeps the per-pixel overlap depth
    of the reference's standard 12k-surfel 256x192 street scene."""
    return math.sqrt((12000.0 / n_surfels) * (256.0 * height) / (192.0 * width))


def make_street_scene(spec: StreetSpec, with_labels: bool = True) -> Tuple[SceneMap, Optional[np.ndarray], Camera]:
    """Returns (scene, labels (N, n_instances) or None, camera)."""
    lib = _lib.load()
    cs = spec.to_c()
    n = C.c_int64()
    cam = A.psm_camera()
    _check(lib.psm_make_street_scene(C.byref(cs), C.byref(n), None, None, None, C.byref(cam)), what="street scene")
    surfels = np.empty((n.value, 13), dtype=np.float64)
    f_sem = np.empty((n.value, spec.c_sem), dtype=np.float64)
    labels = np.empty((n.value, spec.n_instances), dtype=np.float64) if with_labels else None
    _check(lib.psm_make_street_scene(C.byref(cs), C.byref(n), surfels.ctypes.data_as(C.c_void_p),
                                     f_sem.ctypes.data_as(C.c_void_p) if spec.c_sem > 0 else None,
                                     labels.ctypes.data_as(C.c_void_p) if labels is not None else None,
                                     C.byref(cam)), what="street scene")
    return SceneMap(surfels, f_sem), labels, Camera.from_c(cam)


def street_f_ins(spec: StreetSpec) -> np.ndarray:
    """Surfel::f_ins of make_street_scene (N, 8): the 0.3 N(0,1) draws the generator makes
    for every surfel (synthetic.cpp:283-284), for assign_labels."""
    lib = _lib.load()
    cs = spec.to_c()
    n = C.c_int64()
    _check(lib.psm_make_street_scene_ins(C.byref(cs), C.byref(n), None), what="street f_ins")
    f = np.empty((n.value, 8), dtype=np.float64)
    _check(lib.psm_make_street_scene_ins(C.byref(cs), C.byref(n), f.ctypes.data_as(C.c_void_p)), what="street f_ins")
    return f


def trajectory_cameras(n_views: int, width: int, height: int, first: int = 0, count: Optional[int] = None,
                       total: int = 256) -> List[Camera]:
    """C5 views i in [first, first+count) of a closed-form `total`-view trajectory:
    eye = (0.8 sin(2 pi i/T), 0.2 sin(4 pi i/T), 0.05 i), theta = 0.15 sin(2 pi i/T),
    target = eye + 20 (sin theta, 0, cos theta), up (0,-1,0), f = 0.8 W, near 0.1, far 200."""
    count = n_views if count is None else count
    cams = []
    for i in range(first, first + count):
        a = 2.0 * math.pi * (i % total) / total
        eye = (0.8 * math.sin(a), 0.2 * math.sin(2.0 * a), 0.05 * (i % total))
        th = 0.15 * math.sin(a)
        target = (eye[0] + 20.0 * math.sin(th), eye[1], eye[2] + 20.0 * math.cos(th))
        cams.append(Camera.look_at(eye, target, (0.0, -1.0, 0.0), 0.8 * width, 0.8 * width, width, height, 0.1,
                                   200.0))
    return cams
