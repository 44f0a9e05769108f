"""Host-side mirror of the reference render API over the C-ABI.

Names, argument meaning and error behaviour follow proj/include/psimap/raster.hpp
(RasterConfig :42-54, RenderTargets :56-66, render/render_into :142-148,
BenchRow/BenchReport/bench_render :150-172) and core_types.hpp (Camera :36-53,
Camera::make / look_at core_types.cpp:18-60). Planes are numpy arrays shaped
(H, W, C) in the reference's HWC channel-fastest layout, computed on the GPU
in fp32/int32. Errors raise the exception type the reference throws
(ValueError for std::invalid_argument, RuntimeError otherwise).

Every render goes through the CUDA library; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _abi as A
from . import _lib


class Binning(enum.IntEnum):
    Circle = A.BIN_CIRCLE
    Aabb = A.BIN_AABB
    Ellipse = A.BIN_ELLIPSE  # exact support-ellipse vs tile test (north-star Precise Tile Intersection)


class Blending(enum.IntEnum):
    Full = A.BLEND_FULL
    TopK = A.BLEND_TOPK


class PsmError(RuntimeError):
    pass


def _check(status: int, ctx=None, what: str = "") -> None:
    if status == A.PSM_OK:
        return
    msg = what
    if ctx is not None:
        lib = _lib.load()
        m = lib.psm_last_error(ctx)
        if m:
            msg = f"{what}: {m.decode()}" if what else m.decode()
    if status == A.PSM_EINVAL:
        raise ValueError(msg or "invalid argument")
    if status == A.PSM_ENOMEM:
        raise MemoryError(msg or "device allocation failed")
    if status == A.PSM_EUNSUPPORTED:
        raise NotImplementedError(msg or "unsupported on the GPU path")
    raise PsmError(msg or f"CUDA error (status {status})")


@dataclass
class RasterConfig:  # raster.hpp:42-54
    tile_size: int = 16
    chi2: float = 9.0
    alpha_min: float = 1.0 / 255.0
    t_min: float = 1e-4
    support_cutoff: bool = True
    binning: Binning = Binning.Aabb
    blending: Blending = Blending.Full
    top_k: int = 16
    background: tuple = (0.0, 0.0, 0.0)
    render_depth_normal: bool = True
    threads: int = 0

    def to_c(self) -> A.psm_raster_config:
        c = A.psm_raster_config()
        c.tile_size = int(self.tile_size)
        c.chi2 = float(self.chi2)
        c.alpha_min = float(self.alpha_min)
        c.t_min = float(self.t_min)
        c.support_cutoff = int(bool(self.support_cutoff))
        c.binning = int(self.binning)
        c.blending = int(self.blending)
        c.top_k = int(self.top_k)
        for i in range(3):
            c.background[i] = float(self.background[i])
        c.render_depth_normal = int(bool(self.render_depth_normal))
        c.threads = int(self.threads)
        return c


@dataclass
class Camera:  # core_types.hpp:36-53
    r_cw: np.ndarray = field(default_factory=lambda: np.eye(3))
    t_cw: np.ndarray = field(default_factory=lambda: np.zeros(3))
    fx: float = 1.0
    fy: float = 1.0
    cx: float = 0.0
    cy: float = 0.0
    width: int = 0
    height: int = 0
    near_clip: float = 0.01
    far_clip: float = 100.0

    @staticmethod
    def make(r_cw, t_cw, fx, fy, cx, cy, width, height, near_clip, far_clip) -> "Camera":
        lib = _lib.load()
        r = (C.c_double * 9)(*np.asarray(r_cw, dtype=np.float64).reshape(3, 3).T.reshape(-1))  # column-major
        t = (C.c_double * 3)(*np.asarray(t_cw, dtype=np.float64).reshape(3))
        out = A.psm_camera()
        _check(lib.psm_camera_make(C.byref(r), C.byref(t), fx, fy, cx, cy, width, height, near_clip, far_clip,
                                   C.byref(out)), what="camera")
        return Camera.from_c(out)

    @staticmethod
    def look_at(eye, target, up, fx, fy, width, height, near_clip, far_clip) -> "Camera":
        lib = _lib.load()
        e = (C.c_double * 3)(*map(float, eye))
        t = (C.c_double * 3)(*map(float, target))
        u = (C.c_double * 3)(*map(float, up))
        out = A.psm_camera()
        _check(lib.psm_camera_look_at(C.byref(e), C.byref(t), C.byref(u), fx, fy, width, height, near_clip,
                                      far_clip, C.byref(out)), what="camera")
        return Camera.from_c(out)

    @staticmethod
    def from_c(c: A.psm_camera) -> "Camera":
        r = np.array(list(c.r_cw), dtype=np.float64).reshape(3, 3).T  # stored column-major
        return Camera(r, np.array(list(c.t_cw)), c.fx, c.fy, c.cx, c.cy, c.width, c.height, c.near_clip, c.far_clip)

    def to_c(self) -> A.psm_camera:
        c = A.psm_camera()
        r = np.asarray(self.r_cw, dtype=np.float64).reshape(3, 3)
        for col in range(3):
            for row in range(3):
                c.r_cw[col * 3 + row] = float(r[row, col])
        for i in range(3):
            c.t_cw[i] = float(self.t_cw[i])
        c.fx, c.fy, c.cx, c.cy = float(self.fx), float(self.fy), float(self.cx), float(self.cy)
        c.width, c.height = int(self.width), int(self.height)
        c.near_clip, c.far_clip = float(self.near_clip), float(self.far_clip)
        return c


class SceneMap:
    """The render-relevant part of psimap::SceneMap (core_types.hpp:102-111):
    surfels as an (N, 13) fp64 array [center3, quat(w,x,y,z)4, scales2, opacity, color3]
    (Surfel, core_types.hpp:17-25) and f_sem as (N, C_sem) fp64."""

    def __init__(self, surfels13: np.ndarray, f_sem: Optional[np.ndarray] = None,
                 f_ins: Optional[np.ndarray] = None, queries=None):
        self.surfels = np.ascontiguousarray(np.asarray(surfels13, dtype=np.float64).reshape(-1, 13))
        n = self.surfels.shape[0]
        f = np.zeros((n, 0)) if f_sem is None else np.asarray(f_sem, dtype=np.float64)
        if n == 0:
            f = f.reshape(0, f.shape[-1] if f.ndim == 2 else 0)
        self.f_sem = np.ascontiguousarray(f.reshape(n, -1) if n else f)
        # Surfel::f_ins (N, C_ins) and SceneMap::queries (core_types.hpp:105): the panoptic layer's inputs
        self.f_ins = None if f_ins is None else np.ascontiguousarray(np.asarray(f_ins, dtype=np.float64).reshape(n, -1))
        self.queries = list(queries) if queries is not None else []

    def __len__(self) -> int:
        return self.surfels.shape[0]

    def c_sem(self) -> int:  # taken from the first surfel, like SceneMap::c_sem (core_types.hpp:108)
        return 0 if len(self) == 0 else self.f_sem.shape[1]


@dataclass
class RenderTargets:  # raster.hpp:56-66 (fp32 / int32 planes, HWC)
    color: Optional[np.ndarray] = None
    depth: Optional[np.ndarray] = None
    normal: Optional[np.ndarray] = None
    sem_feat: Optional[np.ndarray] = None
    ins_dist: Optional[np.ndarray] = None
    ins_argmax: Optional[np.ndarray] = None
    alpha_acc: Optional[np.ndarray] = None
    blend_count: Optional[np.ndarray] = None
    blended_total: int = 0
    rn_total: int = 0
    rn_per_tile: float = 0.0
    n_proj: int = 0

    def ensure(self, w: int, h: int, c_sem: int, n_q: int) -> None:
        """reset_plane semantics (raster.cpp:255-262): reallocate only on shape change."""
        def want(name, c, dt):
            cur = getattr(self, name)
            if cur is None or cur.shape != (h, w, c) or cur.dtype != dt:
                setattr(self, name, np.zeros((h, w, c), dtype=dt))
        want("color", 3, np.float32)
        want("depth", 2, np.float32)
        want("normal", 3, np.float32)
        want("sem_feat", c_sem, np.float32)
        want("ins_dist", n_q, np.float32)
        want("ins_argmax", 1, np.int32)
        want("alpha_acc", 1, np.float32)
        want("blend_count", 1, np.int32)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None or a.size == 0 else a.ctypes.data_as(C.c_void_p)


class DeviceScene:
    """A scene resident on one GPU (psm_scene_upload)."""

    def __init__(self, renderer: "Renderer", scene: SceneMap, labels: Optional[np.ndarray], exact: bool = False):
        self._r = renderer
        lib = _lib.load()
        n = len(scene)
        lab = None
        n_q = 0
        if labels is not None:
            # MatX N_q x N, column per surfel == (N, N_q) row-major here
            lab = np.ascontiguousarray(np.asarray(labels, dtype=np.float64))
            if lab.ndim != 2 or lab.shape[0] != n:
                raise ValueError("labels must be (N, N_q): one distribution per surfel")
            n_q = lab.shape[1]
        self.handle = C.c_void_p()
        f_ins = getattr(scene, "f_ins", None)
        c_ins = 0 if f_ins is None else f_ins.shape[1]
        desc = A.psm_scene_desc(_ptr(scene.surfels), n, _ptr(scene.f_sem), scene.c_sem(), _ptr(lab), n_q,
                                _ptr(f_ins), c_ins, A.PSM_SCENE_EXACT_FEATURES if exact else 0)
        _check(lib.psm_scene_create(renderer.ctx, C.byref(desc), C.byref(self.handle)), renderer.ctx, "scene upload")
        self.n, self.c_sem, self.n_q = n, (scene.c_sem() if n else 0), (n_q if lab is not None else 0)
        self.c_ins = c_ins
        self.exact = exact

    def free(self) -> None:
        if self.handle:
            _lib.load().psm_scene_free(self._r.ctx, self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Renderer:
    """One psm_ctx on one device: owns a stream and grow-only scratch."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        lib = _lib.load()
        self.ctx = C.c_void_p()
        st = lib.psm_create(device, C.c_void_p(stream) if stream else None, C.byref(self.ctx))
        if st != A.PSM_OK:
            raise PsmError(f"psm_create(device={device}) failed with status {st} (no CUDA device?)")
        self.device = device

    def close(self) -> None:
        if self.ctx:
            _lib.load().psm_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload(self, scene: SceneMap, labels: Optional[np.ndarray] = None, exact: bool = False) -> DeviceScene:
        """psm_scene_create. exact=True also keeps fp64 features/labels on the device
        (render_panoptic reproduces the reference's argmaxes bit for bit)."""
        return DeviceScene(self, scene, labels, exact)

    def assign_labels(self, dscene: DeviceScene, queries, outputs: bool = True):
        """assign_labels (panoptic.cpp:36-91) on the GPU: the scene's label channels become
        the per-surfel distribution over `queries`. Returns (dist (N, Q), argmax (N,)); with
        outputs=False nothing is copied back and the call is asynchronous on the context stream."""
        from .panoptic import pack_queries
        lib = _lib.load()
        feat, mean, cov, alive, cls = pack_queries(queries, dscene.c_ins)
        q = len(queries)
        qs = A.psm_queries(q, dscene.c_ins, _ptr(feat), _ptr(mean), _ptr(cov), _ptr(alive), _ptr(cls))
        dist = np.zeros((dscene.n, q)) if outputs else None
        arg = np.full(dscene.n, -1, np.int32) if outputs else None
        _check(lib.psm_assign_labels(self.ctx, dscene.handle, C.byref(qs), _ptr(dist), _ptr(arg)), self.ctx,
               "assign_labels")
        dscene.n_q = q
        return (dist, arg) if outputs else None

    def render_panoptic_device(self, dscene: DeviceScene, cam: Camera, cfg: RasterConfig, query_class: np.ndarray,
                               planes: dict, counters: bool = False):
        """render_panoptic into device int32 planes {"ids", "classes", "sem_classes": device pointer};
        asynchronous unless counters are asked for."""
        lib = _lib.load()
        qc = np.ascontiguousarray(np.asarray(query_class, dtype=np.int32))
        pt = A.psm_panoptic_targets(planes.get("ids"), planes.get("classes"), planes.get("sem_classes"), 1)
        cnt = A.psm_counters()
        c_cam, c_cfg = cam.to_c(), cfg.to_c()
        _check(lib.psm_render_panoptic(self.ctx, dscene.handle, C.byref(c_cam), C.byref(c_cfg), _ptr(qc), qc.size,
                                       C.byref(pt), C.byref(cnt) if counters else None), self.ctx, "render_panoptic")
        return cnt if counters else None

    def render_panoptic(self, dscene: DeviceScene, cam: Camera, cfg: RasterConfig, query_class,
                        counters: bool = False, out=None):
        """render_panoptic (metrics.cpp:339-369) over a DeviceScene whose labels are assigned
        (assign_labels or uploaded): PanopticRender of (H, W, 1) int32 planes. `out` (a
        PanopticRender of matching shape, e.g. over pinned memory) is reused when given."""
        from .panoptic import PanopticRender
        lib = _lib.load()
        h, w = cam.height, cam.width
        if out is not None and out.ids.shape == (h, w, 1):
            ids, classes, sem = out.ids, out.classes, out.sem_classes
        else:
            ids = np.empty((h, w, 1), np.int32)
            classes = np.empty((h, w, 1), np.int32)
            sem = np.empty((h, w, 1), np.int32)
        qc = np.ascontiguousarray(np.asarray(list(query_class), dtype=np.int32))
        pt = A.psm_panoptic_targets(_ptr(ids), _ptr(classes), _ptr(sem), 0)
        cnt = A.psm_counters()
        c_cam, c_cfg = cam.to_c(), cfg.to_c()
        _check(lib.psm_render_panoptic(self.ctx, dscene.handle, C.byref(c_cam), C.byref(c_cfg), _ptr(qc), qc.size,
                                       C.byref(pt), C.byref(cnt)), self.ctx, "render_panoptic")
        out = PanopticRender(ids, classes, sem)
        return (out, cnt) if counters else out

    def render_panoptic_scene(self, scene: SceneMap, cam: Camera, cfg: RasterConfig):
        """psimap::render_panoptic(scene, cam, cfg): assign_labels over scene.queries, render,
        epilogue, all on the GPU."""
        ds = DeviceScene(self, scene, None, exact=True)
        if scene.queries:
            self.assign_labels(ds, scene.queries)
        return self.render_panoptic(ds, cam, cfg, [q.class_id for q in scene.queries])

    def set_profiling(self, on: bool) -> None:
        _lib.load().psm_set_profiling(self.ctx, int(on))

    def stage_times(self) -> dict:
        t = A.psm_stage_times()
        _lib.load().psm_get_stage_times(self.ctx, C.byref(t))
        return t.as_dict()

    def render_into(self, out: RenderTargets, scene, labels, cam: Camera, cfg: RasterConfig, debug=None) -> RenderTargets:
        """render_into (raster.cpp:273-511) into host planes. `scene` is a SceneMap
        (uploaded for this call, like the reference's per-call borrow) or a DeviceScene."""
        lib = _lib.load()
        ds = scene if isinstance(scene, DeviceScene) else DeviceScene(self, scene, labels)
        out.ensure(cam.width, cam.height, ds.c_sem, ds.n_q)
        tg = A.psm_targets(_ptr(out.color), _ptr(out.depth), _ptr(out.normal), _ptr(out.sem_feat),
                           _ptr(out.ins_dist), _ptr(out.ins_argmax), _ptr(out.alpha_acc), _ptr(out.blend_count), 0)
        cnt = A.psm_counters()
        c_cam, c_cfg = cam.to_c(), cfg.to_c()
        if debug is None:
            st = lib.psm_render(self.ctx, ds.handle, C.byref(c_cam), C.byref(c_cfg), C.byref(tg), C.byref(cnt))
        else:
            st = lib.psm_render_debug(self.ctx, ds.handle, C.byref(c_cam), C.byref(c_cfg), C.byref(tg),
                                      C.byref(cnt), C.byref(debug))
        _check(st, self.ctx, "render")
        out.blended_total = int(cnt.blended_total)
        out.rn_total = int(cnt.rn_total)
        out.rn_per_tile = float(cnt.rn_per_tile)
        out.n_proj = int(cnt.n_proj)
        return out

    def render(self, scene, labels, cam: Camera, cfg: RasterConfig) -> RenderTargets:
        return self.render_into(RenderTargets(), scene, labels, cam, cfg)

    def render_device(self, dscene: DeviceScene, cam: Camera, cfg: RasterConfig, planes: dict,
                      counters: bool = False) -> Optional[A.psm_counters]:
        """Asynchronous render into device planes given as {name: device pointer (int)} on the
        context stream (names as psm_targets). Returns counters (synchronising) if asked."""
        lib = _lib.load()
        tg = A.psm_targets(*(planes.get(k) for k in ("color", "depth", "normal", "sem_feat", "ins_dist",
                                                      "ins_argmax", "alpha_acc", "blend_count")), 1)
        c_cam, c_cfg = cam.to_c(), cfg.to_c()
        cnt = A.psm_counters()
        st = lib.psm_render(self.ctx, dscene.handle, C.byref(c_cam), C.byref(c_cfg), C.byref(tg),
                            C.byref(cnt) if counters else None)
        _check(st, self.ctx, "render")
        return cnt if counters else None

    def render_batch_device(self, dscene: DeviceScene, cams: Sequence[Camera], cfg: RasterConfig,
                            planes: Sequence[dict]) -> None:
        """psm_render_batch into device planes (one {name: device pointer} dict per view, as
        render_device): asynchronous and pipelined over two streams; psm_sync (`sync`) validates."""
        lib = _lib.load()
        n = len(cams)
        if len(planes) != n:
            raise ValueError("one plane set per camera")
        tg = (A.psm_targets * max(n, 1))()
        for i, pl in enumerate(planes):
            tg[i] = A.psm_targets(*(pl.get(k) for k in ("color", "depth", "normal", "sem_feat", "ins_dist",
                                                        "ins_argmax", "alpha_acc", "blend_count")), 1)
        cc = (A.psm_camera * max(n, 1))(*(c.to_c() for c in cams))
        c_cfg = cfg.to_c()
        _check(lib.psm_render_batch(self.ctx, dscene.handle, cc, n, C.byref(c_cfg), tg, None), self.ctx,
               "render_batch")

    def render_backward(self, scene, labels, cam: Camera, cfg: RasterConfig, g_color=None, g_sem=None,
                        g_ins=None) -> dict:
        """The render backward (pipeline.cpp:347-486) on the GPU: gradients of
        L = <g_color, colour> + <g_sem, sem_feat> + <g_ins, ins_dist> w.r.t. every surfel parameter
        (opacity, color, f_sem, labels, center, rotation, scales). `scene` is a SceneMap or a
        DeviceScene (exact=True keeps the feature dot products in fp64)."""
        lib = _lib.load()
        ds = scene if isinstance(scene, DeviceScene) else DeviceScene(self, scene, labels, exact=True)
        n = ds.n
        gp = [None if a is None else np.ascontiguousarray(a, dtype=np.float64) for a in (g_color, g_sem, g_ins)]
        out = {"opacity": np.zeros(n), "color": np.zeros((n, 3)), "f_sem": np.zeros((n, ds.c_sem)),
               "labels": np.zeros((n, ds.n_q)), "center": np.zeros((n, 3)), "rotation": np.zeros((n, 4)),
               "scales": np.zeros((n, 2))}
        pg = A.psm_plane_grads(*[_ptr(a) for a in gp])
        sg = A.psm_scene_grads(*[_ptr(out[k]) for k in ("opacity", "color", "f_sem", "labels", "center", "rotation",
                                                          "scales")])
        c_cam, c_cfg = cam.to_c(), cfg.to_c()
        _check(lib.psm_render_backward(self.ctx, ds.handle, C.byref(c_cam), C.byref(c_cfg), C.byref(pg), C.byref(sg)),
               self.ctx, "render_backward")
        return out

    def sync(self) -> A.psm_counters:
        lib = _lib.load()
        _check(lib.psm_sync(self.ctx), self.ctx, "sync")
        cnt = A.psm_counters()
        lib.psm_last_counters(self.ctx, C.byref(cnt))
        return cnt


@dataclass
class BenchRow:  # raster.hpp:150-160
    name: str
    binning: Binning
    blending: Blending
    time_ms: float = 0.0
    fps: float = 0.0
    rn_total: int = 0
    rn_per_tile: float = 0.0
    blended_total: int = 0
    blended_per_pixel: float = 0.0


@dataclass
class BenchReport:  # raster.hpp:162-167
    rows: List[BenchRow] = field(default_factory=list)
    repetitions: int = 0
    width: int = 0
    height: int = 0
    surfel_count: int = 0


_default: Optional[Renderer] = None


def default_renderer() -> Renderer:
    global _default
    if _default is None:
        _default = Renderer(0)
    return _default


def render(scene, labels, cam: Camera, cfg: RasterConfig) -> RenderTargets:
    return default_renderer().render(scene, labels, cam, cfg)


def render_into(out: RenderTargets, scene, labels, cam: Camera, cfg: RasterConfig) -> RenderTargets:
    return default_renderer().render_into(out, scene, labels, cam, cfg)


def bench_render(scene, labels, cam: Camera, repetitions: int, base_cfg: RasterConfig,
                 renderer: Optional[Renderer] = None, binnings=None) -> BenchReport:
    """The 4-row ablation grid of bench_render (raster.cpp:513-573): baseline
    (Circle+Full), precise_tile (Aabb+Full), topk (Circle+TopK), full_method
    (Aabb+TopK). One warm-up, `repetitions` timed renders, min time. Times are
    CUDA-event device times of the whole render (K1..K7) with device-resident
    targets; counters come from the timed frames. `binnings` may override the
    precise binning (e.g. Binning.Ellipse)."""
    import torch  # device planes for the timed renders (plumbing only)

    r = renderer or default_renderer()
    ds = scene if isinstance(scene, DeviceScene) else r.upload(scene, labels)
    precise = Binning.Aabb if binnings is None else binnings
    rows = [("baseline", Binning.Circle, Blending.Full), ("precise_tile", precise, Blending.Full),
            ("topk", Binning.Circle, Blending.TopK), ("full_method", precise, Blending.TopK)]
    w, h = cam.width, cam.height
    dev = torch.device("cuda", r.device)
    planes = {
        "color": torch.empty(h * w * 3, dtype=torch.float32, device=dev),
        "depth": torch.empty(h * w * 2, dtype=torch.float32, device=dev),
        "normal": torch.empty(h * w * 3, dtype=torch.float32, device=dev),
        "sem_feat": torch.empty(max(h * w * ds.c_sem, 1), dtype=torch.float32, device=dev),
        "ins_dist": torch.empty(max(h * w * ds.n_q, 1), dtype=torch.float32, device=dev),
        "ins_argmax": torch.empty(h * w, dtype=torch.int32, device=dev),
        "alpha_acc": torch.empty(h * w, dtype=torch.float32, device=dev),
        "blend_count": torch.empty(h * w, dtype=torch.int32, device=dev),
    }
    ptrs = {k: v.data_ptr() for k, v in planes.items()}
    rep = BenchReport(repetitions=repetitions, width=w, height=h, surfel_count=ds.n)
    r.set_profiling(True)
    try:
        for name, binning, blending in rows:
            cfg = RasterConfig(**{**base_cfg.__dict__, "binning": binning, "blending": blending})
            r.render_device(ds, cam, cfg, ptrs, counters=True)  # warm-up
            best = math.inf
            cnt = None
            for _ in range(max(repetitions, 1)):
                cnt = r.render_device(ds, cam, cfg, ptrs, counters=True)
                best = min(best, r.stage_times()["total"])
            row = BenchRow(name, binning, blending, time_ms=best, fps=1000.0 / best if best > 0 else 0.0,
                           rn_total=int(cnt.rn_total), rn_per_tile=float(cnt.rn_per_tile),
                           blended_total=int(cnt.blended_total),
                           blended_per_pixel=float(cnt.blended_total) / (w * h))
            rep.rows.append(row)
    finally:
        r.set_profiling(False)
    return rep
