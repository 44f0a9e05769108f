"""The reference's stage functions and RenderCache on the GPU (include/psm.h "Stage entry
points"), with the reference's names and argument meaning (proj/include/psimap/raster.hpp:21-126):

  project_surfel(s, cam, cfg)            -> ProjectedSurfel or None       raster.cpp:94-142
  bin_circle(projected, cam, cfg)        -> TileGrid                      raster.cpp:144-147
  bin_aabb(projected, cam, cfg, chi2)    -> TileGrid                      raster.cpp:149-152
  sample_surfel_alpha(proj, cam, px, py, cfg) -> AlphaSample              raster.cpp:154-169
  evaluate_alpha(proj, s, cam, px, py, cfg)   -> float                    raster.cpp:171-177
  topk_select(keys, k)                   -> selected flags                raster.cpp:225-251
  render(..., cache=RenderCache())       fills RenderCache                raster.cpp:310-315,399-403

Batch forms (project_surfels, sample_alpha, topk_select_lists) take many inputs per device
call. Every call runs on the device through libpsm.so; results are the reference's bits.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _abi as A
from . import _lib
from .raster import Binning, Camera, DeviceScene, RasterConfig, Renderer, RenderTargets, _check, _ptr, default_renderer


@dataclass
class ProjectedSurfel:  # raster.hpp:21-30
    source: int
    screen_center: np.ndarray
    sigma: np.ndarray
    sort_depth: float
    h: np.ndarray
    h_inv: np.ndarray
    footprint_inv: np.ndarray
    normal_vis: np.ndarray

    @staticmethod
    def from_c(p: A.psm_projected) -> "ProjectedSurfel":
        col = lambda a, n: np.array(list(a)).reshape(n, n).T  # column-major -> (row, col)
        return ProjectedSurfel(int(p.source), np.array(list(p.screen_center)), col(p.sigma, 2), float(p.sort_depth),
                               col(p.h, 3), col(p.h_inv, 3), col(p.footprint_inv, 2), np.array(list(p.normal_vis)))

    def to_c(self) -> A.psm_projected:
        p = A.psm_projected()
        p.source = self.source
        flat = lambda m: list(np.asarray(m, dtype=np.float64).T.reshape(-1))
        p.screen_center[:] = list(self.screen_center)
        p.sigma[:] = flat(self.sigma)
        p.sort_depth = self.sort_depth
        p.h[:] = flat(self.h)
        p.h_inv[:] = flat(self.h_inv)
        p.footprint_inv[:] = flat(self.footprint_inv)
        p.normal_vis[:] = list(self.normal_vis)
        return p


@dataclass
class TileGrid:  # raster.hpp:32-40
    tile_size: int = 16
    tiles_x: int = 0
    tiles_y: int = 0
    tiles: List[np.ndarray] = field(default_factory=list)  # projected indices, ascending (depth, source)
    rn_total: int = 0
    rn_per_tile: float = 0.0

    def tile_count(self) -> int:
        return self.tiles_x * self.tiles_y


@dataclass
class AlphaSample:  # raster.hpp:103-108
    alpha: float = 0.0
    u: float = 0.0
    v: float = 0.0
    w2: float = 0.0
    inside: bool = False


@dataclass
class RenderCache:  # raster.hpp:76-82
    projected: List[ProjectedSurfel] = field(default_factory=list)
    grid: Optional[TileGrid] = None
    pixel_offsets: Optional[np.ndarray] = None  # (W*H+1,) CSR over `contribs` (RenderCache::pixels)
    contribs: Optional[np.ndarray] = None       # structured (proj, alpha, u, v), blend order per pixel
    cfg: Optional[RasterConfig] = None
    width: int = 0
    height: int = 0

    def pixel(self, x: int, y: int) -> np.ndarray:
        i = y * self.width + x
        return self.contribs[self.pixel_offsets[i]:self.pixel_offsets[i + 1]]


CONTRIB_DTYPE = np.dtype([("proj", np.int32), ("pad", np.int32), ("alpha", np.float64), ("u", np.float64),
                          ("v", np.float64)])


def _r(renderer: Optional[Renderer]) -> Renderer:
    return renderer or default_renderer()


def project_surfels(surfels13, cam: Camera, cfg: RasterConfig, renderer: Optional[Renderer] = None):
    """project_surfel over every row of an (N, 13) array: (ctypes psm_projected array, status (N,) int32:
    1 projected / 0 culled). Raises ValueError on a degenerate quaternion (std::invalid_argument)."""
    r = _r(renderer)
    s = np.ascontiguousarray(np.asarray(surfels13, dtype=np.float64).reshape(-1, 13))
    n = s.shape[0]
    out = (A.psm_projected * max(n, 1))()
    status = np.zeros(n, np.int32)
    bad = C.c_int64(-1)
    _check(_lib.load().psm_project_surfels(r.ctx, _ptr(s), n, C.byref(cam.to_c()), C.byref(cfg.to_c()), out,
                                           _ptr(status), C.byref(bad)), r.ctx, "project_surfel")
    return out, status


def project_surfel(surfel13, cam: Camera, cfg: RasterConfig,
                   renderer: Optional[Renderer] = None) -> Optional[ProjectedSurfel]:
    """project_surfel (raster.cpp:94-142): None when culled; source = -1 (the caller fills it)."""
    out, status = project_surfels(np.asarray(surfel13).reshape(1, 13), cam, cfg, renderer)
    return ProjectedSurfel.from_c(out[0]) if status[0] else None


def _projected_array(projected: Sequence) -> "C.Array":
    if isinstance(projected, C.Array):
        return projected
    arr = (A.psm_projected * max(len(projected), 1))()
    for i, p in enumerate(projected):
        arr[i] = p.to_c() if isinstance(p, ProjectedSurfel) else p
    return arr


def _bin(projected, cam: Camera, cfg: RasterConfig, binning: int, chi2: float, renderer) -> TileGrid:
    r = _r(renderer)
    lib = _lib.load()
    arr = _projected_array(projected)
    n = len(projected)
    ts = cfg.tile_size
    tx, ty = (cam.width + ts - 1) // ts, (cam.height + ts - 1) // ts
    counts = np.zeros(tx * ty, np.int32)
    cnt = A.psm_counters()
    c_cam, c_cfg = cam.to_c(), cfg.to_c()
    _check(lib.psm_bin_projected(r.ctx, arr, n, C.byref(c_cam), C.byref(c_cfg), binning, chi2, _ptr(counts), None, 0,
                                 C.byref(cnt)), r.ctx, "bin")
    total = int(cnt.rn_total)
    lists = np.zeros(max(total, 1), np.int32)
    if total:
        _check(lib.psm_bin_projected(r.ctx, arr, n, C.byref(c_cam), C.byref(c_cfg), binning, chi2, _ptr(counts),
                                     _ptr(lists), total, C.byref(cnt)), r.ctx, "bin")
    offs = np.concatenate([[0], np.cumsum(counts)])
    return TileGrid(ts, tx, ty, [lists[offs[t]:offs[t + 1]].copy() for t in range(tx * ty)], total,
                    float(cnt.rn_per_tile))


def bin_circle(projected, cam: Camera, cfg: RasterConfig, renderer: Optional[Renderer] = None) -> TileGrid:
    """bin_circle (raster.cpp:144-147): every tile of the bounding square of the chi2 circle."""
    return _bin(projected, cam, cfg, A.BIN_CIRCLE, cfg.chi2, renderer)


def bin_aabb(projected, cam: Camera, cfg: RasterConfig, chi2: float, renderer: Optional[Renderer] = None) -> TileGrid:
    """bin_aabb (raster.cpp:149-152): every tile of [cx +- sqrt(chi2 F00)] x [cy +- sqrt(chi2 F11)]."""
    return _bin(projected, cam, cfg, A.BIN_AABB, chi2, renderer)


def sample_alpha(projected, opacity, proj_index, px, py, cam: Camera, cfg: RasterConfig,
                 renderer: Optional[Renderer] = None) -> np.ndarray:
    """Batched sample_surfel_alpha + evaluate_alpha: structured array (alpha, u, v, w2, inside) per query."""
    r = _r(renderer)
    arr = _projected_array(projected)
    op = np.ascontiguousarray(np.asarray(opacity, dtype=np.float64))
    idx = np.ascontiguousarray(np.asarray(proj_index, dtype=np.int32))
    x = np.ascontiguousarray(np.asarray(px, dtype=np.float64))
    y = np.ascontiguousarray(np.asarray(py, dtype=np.float64))
    m = idx.size
    out = np.zeros(m, dtype=np.dtype([("alpha", np.float64), ("u", np.float64), ("v", np.float64),
                                      ("w2", np.float64), ("inside", np.int32), ("pad", np.int32)]))
    _check(_lib.load().psm_sample_alpha(r.ctx, arr, _ptr(op), len(projected), _ptr(idx), _ptr(x), _ptr(y), m,
                                        C.byref(cam.to_c()), C.byref(cfg.to_c()), _ptr(out)), r.ctx, "sample_alpha")
    return out


def sample_surfel_alpha(proj: ProjectedSurfel, cam: Camera, px: float, py: float, cfg: RasterConfig,
                        renderer: Optional[Renderer] = None) -> AlphaSample:
    """sample_surfel_alpha (raster.cpp:154-169): AlphaSample.alpha stays 0 as in the reference."""
    o = sample_alpha([proj], [0.0], [0], [px], [py], cam, cfg, renderer)[0]
    return AlphaSample(0.0, float(o["u"]), float(o["v"]), float(o["w2"]), bool(o["inside"]))


def evaluate_alpha(proj: ProjectedSurfel, surfel13, cam: Camera, px: float, py: float, cfg: RasterConfig,
                   renderer: Optional[Renderer] = None) -> float:
    """evaluate_alpha (raster.cpp:171-177) with the surfel's opacity (column 9 of the 13-double row)."""
    op = float(np.asarray(surfel13, dtype=np.float64).reshape(13)[9])
    return float(sample_alpha([proj], [op], [0], [px], [py], cam, cfg, renderer)[0]["alpha"])


def topk_select_lists(weights, proj, offsets, k: int, renderer: Optional[Renderer] = None) -> np.ndarray:
    """topk_select over many lists at once (CSR offsets): boolean selected flags per entry."""
    r = _r(renderer)
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
    p = np.ascontiguousarray(np.asarray(proj, dtype=np.int32))
    o = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
    sel = np.zeros(w.size, np.int8)
    _check(_lib.load().psm_topk_select(r.ctx, _ptr(w), _ptr(p), _ptr(o), o.size - 1, k, _ptr(sel)), r.ctx,
           "topk_select")
    return sel.astype(bool)


def topk_select(weights, proj, k: int, renderer: Optional[Renderer] = None) -> np.ndarray:
    """topk_select (raster.cpp:225-251) of one list of WeightKeys (weight, proj)."""
    return topk_select_lists(weights, proj, [0, len(weights)], k, renderer)


def render_cached(scene, labels, cam: Camera, cfg: RasterConfig, cache: RenderCache,
                  renderer: Optional[Renderer] = None, out: Optional[RenderTargets] = None) -> RenderTargets:
    """render (raster.cpp:266-511) with a RenderCache: the planes, plus the projected surfels, the
    tile grid and every pixel's contributors in blend order (proj index, alpha, u, v)."""
    r = _r(renderer)
    lib = _lib.load()
    ds = scene if isinstance(scene, DeviceScene) else r.upload(scene, labels)
    out = out or RenderTargets()
    out.ensure(cam.width, cam.height, ds.c_sem, ds.n_q)
    tg = A.psm_targets(_ptr(out.color), _ptr(out.depth), _ptr(out.normal), _ptr(out.sem_feat), _ptr(out.ins_dist),
                       _ptr(out.ins_argmax), _ptr(out.alpha_acc), _ptr(out.blend_count), 0)
    cnt = A.psm_counters()
    c_cam, c_cfg = cam.to_c(), cfg.to_c()
    ts = cfg.tile_size
    tiles = ((cam.width + ts - 1) // ts) * ((cam.height + ts - 1) // ts)
    npx = cam.width * cam.height
    co = A.psm_render_cache_out()  # sizing pass
    _check(lib.psm_render_cache(r.ctx, ds.handle, C.byref(c_cam), C.byref(c_cfg), C.byref(tg), C.byref(cnt),
                                C.byref(co)), r.ctx, "render_cache")
    proj = (A.psm_projected * max(co.n_projected, 1))()
    counts = np.zeros(tiles, np.int32)
    lists = np.zeros(max(co.n_tile_entries, 1), np.int32)
    offs = np.zeros(npx + 1, np.int64)
    contribs = np.zeros(max(co.n_contribs, 1), CONTRIB_DTYPE)
    co = A.psm_render_cache_out(C.cast(proj, C.c_void_p), co.n_projected, 0, _ptr(counts), _ptr(lists),
                                co.n_tile_entries, 0, _ptr(offs), _ptr(contribs), co.n_contribs, 0)
    _check(lib.psm_render_cache(r.ctx, ds.handle, C.byref(c_cam), C.byref(c_cfg), C.byref(tg), C.byref(cnt),
                                C.byref(co)), r.ctx, "render_cache")
    out.blended_total = int(cnt.blended_total)
    out.rn_total = int(cnt.rn_total)
    out.rn_per_tile = float(cnt.rn_per_tile)
    out.n_proj = int(cnt.n_proj)
    goffs = np.concatenate([[0], np.cumsum(counts)])
    cache.projected = [ProjectedSurfel.from_c(proj[i]) for i in range(co.n_projected)]
    cache.grid = TileGrid(ts, (cam.width + ts - 1) // ts, (cam.height + ts - 1) // ts,
                          [lists[goffs[t]:goffs[t + 1]].copy() for t in range(tiles)], int(co.n_tile_entries),
                          float(cnt.rn_per_tile))
    cache.pixel_offsets = offs
    cache.contribs = contribs[:co.n_contribs]
    cache.cfg = cfg
    cache.width, cache.height = cam.width, cam.height
    return out
