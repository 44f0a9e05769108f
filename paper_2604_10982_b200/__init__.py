"""B200-native Ψ-Map render hot path: the 2D Gaussian-surfel panoptic rasterizer
(project -> bin -> sort -> composite with Top-K) as hand-written sm_100a kernels
behind a C-ABI (include/psm.h), with a host mirror of psimap::render /
render_into / bench_render (proj/include/psimap/raster.hpp:142-172).
"""
from .raster import (Binning, Blending, BenchReport, BenchRow, Camera, DeviceScene, PsmError, RasterConfig,
                     Renderer, RenderTargets, SceneMap, bench_render, render, render_into)
from .scene import StreetSpec, density_scale, make_street_scene, street_f_ins, trajectory_cameras
from .panoptic import InstanceQuery, PanopticRender, street_queries

__all__ = [
    "Binning", "Blending", "BenchReport", "BenchRow", "Camera", "DeviceScene", "PsmError", "RasterConfig",
    "Renderer", "RenderTargets", "SceneMap", "bench_render", "render", "render_into", "StreetSpec",
    "density_scale", "make_street_scene", "trajectory_cameras", "street_f_ins", "InstanceQuery",
    "PanopticRender", "street_queries",
]
