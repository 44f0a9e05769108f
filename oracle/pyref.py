"""ctypes wrapper of oracle/_ref/libpsimap_ref.so: the REFERENCE'S OWN render path
(/root/reference/proj/src/{raster,math_util,core_types,synthetic}.cpp), the panoptic rows
(panoptic.cpp assign_labels, metrics.cpp render_panoptic) and the backward row (pipeline.cpp
pipeline_backward with losses.cpp / sogmm.cpp, raster.cpp project_surfel_backward), compiled unchanged by
oracle/ref/Makefile against the minimal Eigen stand-in oracle/eigen_min.
TEST INFRASTRUCTURE ONLY: imported by tests/ and by bench.py's reference arm, never by
the product package.

`available()` is False where the library was not built (it needs /root/reference at
build time; the built .so travels to the GPU box with the repo snapshot).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "libpsimap_ref.so")
REF_SRC = "/root/reference/proj/src/raster.cpp"
_lib = None


def _abi():
    # struct layouts of include/psm.h (plain ctypes; importing _abi does not load libpsm.so)
    from paper_2604_10982_b200 import _abi as A
    return A


class ref_projected(C.Structure):
    _fields_ = [("status", C.c_int32), ("center", C.c_double * 2), ("sigma", C.c_double * 4),
                ("sort_depth", C.c_double), ("h", C.c_double * 9), ("h_inv", C.c_double * 9),
                ("finv", C.c_double * 4), ("normal_vis", C.c_double * 3)]


def build() -> bool:
    """Builds oracle/_ref when the reference tree is present (this container only)."""
    if not os.path.exists(REF_SRC):
        return os.path.exists(LIB)
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "ref")], check=True)
    return True


def available() -> bool:
    return os.path.exists(LIB) or os.path.exists(REF_SRC)


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB):
        build()
    A = _abi()
    lib = C.CDLL(LIB)
    vp, P = C.c_void_p, C.POINTER
    sig = {
        "ref_make_street_scene": (C.c_int, [P(A.psm_street_spec), P(C.c_int64), vp, vp, vp, vp, P(A.psm_camera)]),
        "ref_camera_look_at": (C.c_int, [vp, vp, vp, C.c_double, C.c_double, C.c_int32, C.c_int32, C.c_double,
                                         C.c_double, P(A.psm_camera)]),
        "ref_scene_create": (vp, [vp, C.c_int64, vp, C.c_int32, vp, C.c_int32]),
        "ref_scene_free": (None, [vp]),
        "ref_render_into": (C.c_int, [vp, P(A.psm_camera), P(A.psm_raster_config), P(C.c_uint64)]),
        "ref_targets_copy": (None, [vp] * 9),
        "ref_bin": (C.c_int, [vp, P(A.psm_camera), P(A.psm_raster_config), C.c_int32, C.c_double, vp, vp,
                              C.c_int64, P(A.psm_counters)]),
        "ref_project_surfel": (C.c_int, [vp, P(A.psm_camera), P(A.psm_raster_config), P(ref_projected)]),
        "ref_evaluate_alpha": (C.c_double, [vp, P(A.psm_camera), C.c_double, C.c_double, P(A.psm_raster_config),
                                            P(C.c_double), P(C.c_double), P(C.c_double), P(C.c_int32)]),
        "ref_topk_select": (None, [vp, vp, C.c_int32, C.c_int32, vp]),
        "ref_bench_render": (C.c_int, [vp, P(A.psm_camera), C.c_int32, P(A.psm_raster_config), vp]),
        "ref_assign_labels": (C.c_int, [vp, C.c_int64, vp, C.c_int32, C.c_int32, vp, vp, vp, vp, vp, vp]),
        "ref_render_panoptic": (C.c_int, [vp, C.c_int64, vp, C.c_int32, vp, C.c_int32, C.c_int32, vp, vp, vp, vp, vp,
                                          P(A.psm_camera), P(A.psm_raster_config), vp, vp, vp]),
        "ref_panoptic_scene_create": (vp, [vp, C.c_int64, vp, C.c_int32, vp, C.c_int32, C.c_int32, vp, vp, vp, vp,
                                           vp]),
        "ref_panoptic_scene_free": (None, [vp]),
        "ref_render_panoptic_h": (C.c_int, [vp, P(A.psm_camera), P(A.psm_raster_config), vp, vp, vp]),
        "ref_project_surfel_backward": (C.c_int, [vp, P(A.psm_camera), P(A.psm_raster_config), vp, vp, vp, vp]),
        "ref_pipeline_backward": (C.c_int, [vp, P(A.psm_camera), P(A.psm_raster_config), C.c_int32, vp, vp,
                                            C.c_double, C.c_double, C.c_double, C.c_double, P(A.psm_scene_grads),
                                            vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    _lib = lib
    return lib


def _p(a: Optional[np.ndarray]):
    return None if a is None or a.size == 0 else a.ctypes.data_as(C.c_void_p)


def make_street_scene(n_surfels=12000, seed=7, min_aspect=5.0, image_w=256, image_h=192, c_sem=32,
                      n_instances=256, labels=True):
    """make_street_scene (synthetic.cpp:236-312) exactly as the reference generates it:
    (surfels13 (N,13), f_sem (N,C), labels (N,n_instances) or None, f_ins (N,8), psm_camera)."""
    A = _abi()
    lib = load()
    spec = A.psm_street_spec(n_surfels, seed, min_aspect, image_w, image_h, c_sem, n_instances, 1.0)
    n = C.c_int64()
    cam = A.psm_camera()
    if lib.ref_make_street_scene(C.byref(spec), C.byref(n), None, None, None, None, C.byref(cam)) != 0:
        raise ValueError("make_street_scene failed")
    s = np.empty((n.value, 13))
    f = np.empty((n.value, c_sem))
    lab = np.empty((n.value, n_instances)) if labels else None
    fi = np.empty((n.value, 8))
    lib.ref_make_street_scene(C.byref(spec), C.byref(n), _p(s), _p(f), _p(lab), _p(fi), C.byref(cam))
    return s, f, lab, fi, cam


class RefScene:
    """A psimap::SceneMap (+ labels MatX) held by the reference library, rendered with render_into."""

    def __init__(self, surfels13, f_sem=None, labels=None):
        self.lib = load()
        self.surfels = np.ascontiguousarray(np.asarray(surfels13, dtype=np.float64).reshape(-1, 13))
        n = self.surfels.shape[0]
        f = np.zeros((n, 0)) if f_sem is None else np.ascontiguousarray(np.asarray(f_sem, dtype=np.float64))
        self.c_sem = f.shape[1] if n else 0
        lab = None if labels is None else np.ascontiguousarray(np.asarray(labels, dtype=np.float64))
        self.n_q = 0 if lab is None else lab.shape[1]
        self.h = self.lib.ref_scene_create(_p(self.surfels), n, _p(f), self.c_sem, _p(lab), self.n_q)

    def close(self):
        if self.h:
            self.lib.ref_scene_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def render_into(self, cam_c, cfg_c) -> int:
        """One render_into (raster.cpp:273-511); returns blended_total. Raises on a degenerate quaternion."""
        bt = C.c_uint64()
        st = self.lib.ref_render_into(self.h, C.byref(cam_c), C.byref(cfg_c), C.byref(bt))
        if st != 0:
            raise ValueError("degenerate quaternion")
        return int(bt.value)

    def render(self, cam, cfg) -> dict:
        """render (raster.cpp:266-271): fp64 planes (H, W, C) and blended_total."""
        bt = self.render_into(cam.to_c(), cfg.to_c())
        w, h = cam.width, cam.height
        out = {"color": np.zeros((h, w, 3)), "depth": np.zeros((h, w, 2)), "normal": np.zeros((h, w, 3)),
               "sem_feat": np.zeros((h, w, self.c_sem)), "ins_dist": np.zeros((h, w, self.n_q)),
               "ins_argmax": np.zeros((h, w, 1), np.int32), "alpha_acc": np.zeros((h, w, 1)),
               "blend_count": np.zeros((h, w, 1), np.int32)}
        self.lib.ref_targets_copy(self.h, *[_p(out[k]) for k in ("color", "depth", "normal", "sem_feat", "ins_dist",
                                                                  "ins_argmax", "alpha_acc", "blend_count")])
        out["blended_total"] = bt
        return out

    def bin(self, cam, cfg, binning: int, chi2: Optional[float] = None) -> dict:
        """project_surfel + bin_circle / bin_aabb: per-tile source-id lists and TileGrid counters."""
        A = _abi()
        c, k = cam.to_c(), cfg.to_c()
        chi = cfg.chi2 if chi2 is None else chi2
        tiles = ((cam.width + cfg.tile_size - 1) // cfg.tile_size) * ((cam.height + cfg.tile_size - 1) // cfg.tile_size)
        counts = np.zeros(tiles, np.int32)
        cnt = A.psm_counters()
        if self.lib.ref_bin(self.h, C.byref(c), C.byref(k), binning, chi, _p(counts), None, 0, C.byref(cnt)) != 0:
            raise ValueError("degenerate quaternion")
        total = int(counts.sum())
        lists = np.zeros(max(total, 1), np.int32)
        self.lib.ref_bin(self.h, C.byref(c), C.byref(k), binning, chi, None, _p(lists), total, None)
        offs = np.concatenate([[0], np.cumsum(counts)])
        return {"tiles": [lists[offs[t]:offs[t + 1]].copy() for t in range(tiles)], "counts": counts,
                "lists": lists[:total], "rn_total": int(cnt.rn_total), "rn_per_tile": float(cnt.rn_per_tile),
                "n_proj": int(cnt.n_proj)}

    def bench_render(self, cam, reps: int, cfg) -> list:
        """bench_render (raster.cpp:513-573): rows (time_ms, fps, rn_total, rn_per_tile, blended, per_pixel)."""
        rows = np.zeros((4, 6))
        if self.lib.ref_bench_render(self.h, C.byref(cam.to_c()), reps, C.byref(cfg.to_c()), _p(rows)) != 0:
            raise ValueError("degenerate quaternion")
        return rows


    def pipeline_backward(self, cam, cfg, rgb_gt, sem_gt=None, lambda_s=0.2, l_rgb=1.0, l_sem=0.5, l_iso=0.0,
                          smooth=False) -> dict:
        """pipeline_backward (pipeline.cpp:253-600) of this query-free scene with no SOGMM model:
        the surfel gradients (psm_scene_grads fields, per-surfel rows) and "g_color_plane", the colour
        gradient the reference fed its blending backward (loss_rgb_backward, pipeline.cpp:266)."""
        A = _abi()
        n = self.surfels.shape[0]
        out = {"opacity": np.zeros(n), "color": np.zeros((n, 3)), "f_sem": np.zeros((n, self.c_sem)),
               "center": np.zeros((n, 3)), "rotation": np.zeros((n, 4)), "scales": np.zeros((n, 2)),
               "g_color_plane": np.zeros((cam.height, cam.width, 3))}
        sg = A.psm_scene_grads(_p(out["opacity"]), _p(out["color"]), _p(out["f_sem"]), None, _p(out["center"]),
                               _p(out["rotation"]), _p(out["scales"]))
        rgb = np.ascontiguousarray(np.asarray(rgb_gt, dtype=np.float64).reshape(cam.height, cam.width, 3))
        sem = None if sem_gt is None else np.ascontiguousarray(np.asarray(sem_gt, dtype=np.int32).reshape(-1))
        st = self.lib.ref_pipeline_backward(self.h, C.byref(cam.to_c()), C.byref(cfg.to_c()), int(smooth), _p(rgb),
                                            _p(sem), lambda_s, l_rgb, l_sem, l_iso, C.byref(sg),
                                            _p(out["g_color_plane"]))
        if st != 0:
            raise ValueError("degenerate quaternion")
        return out


def project_surfel_backward(s13, cam, cfg, g_hinv) -> Optional[dict]:
    """project_surfel_backward (raster.cpp:179-203) under the surfel's own projection; None if culled."""
    s = np.ascontiguousarray(np.asarray(s13, dtype=np.float64).reshape(13))
    g = np.ascontiguousarray(np.asarray(g_hinv, dtype=np.float64).reshape(3, 3))
    dc, dq, ds = np.zeros(3), np.zeros(4), np.zeros(2)
    st = load().ref_project_surfel_backward(_p(s), C.byref(cam.to_c()), C.byref(cfg.to_c()), _p(g), _p(dc), _p(dq),
                                            _p(ds))
    if st < 0:
        raise ValueError("degenerate quaternion")
    return None if st == 0 else {"center": dc, "rotation": dq, "scales": ds}


def project_surfel(s13, cam, cfg) -> Optional[dict]:
    s = np.ascontiguousarray(np.asarray(s13, dtype=np.float64).reshape(13))
    out = ref_projected()
    st = load().ref_project_surfel(_p(s), C.byref(cam.to_c()), C.byref(cfg.to_c()), C.byref(out))
    if st < 0:
        raise ValueError("degenerate quaternion")
    if st == 0:
        return None
    return {"center": np.array(list(out.center)), "sigma": np.array(list(out.sigma)).reshape(2, 2).T,
            "sort_depth": out.sort_depth, "h": np.array(list(out.h)).reshape(3, 3).T,
            "h_inv": np.array(list(out.h_inv)).reshape(3, 3).T,
            "footprint_inv": np.array(list(out.finv)).reshape(2, 2).T, "normal_vis": np.array(list(out.normal_vis))}


def evaluate_alpha(s13, cam, px, py, cfg) -> dict:
    s = np.ascontiguousarray(np.asarray(s13, dtype=np.float64).reshape(13))
    u, v, w2, inside = C.c_double(), C.c_double(), C.c_double(), C.c_int32()
    a = load().ref_evaluate_alpha(_p(s), C.byref(cam.to_c()), px, py, C.byref(cfg.to_c()), C.byref(u), C.byref(v),
                                  C.byref(w2), C.byref(inside))
    return {"alpha": a, "u": u.value, "v": v.value, "w2": w2.value, "inside": bool(inside.value)}


def topk_select(weights, proj, k: int) -> np.ndarray:
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
    p = np.ascontiguousarray(np.asarray(proj, dtype=np.int32))
    sel = np.zeros(len(w), dtype=np.int8)
    load().ref_topk_select(_p(w), _p(p), len(w), k, _p(sel))
    return sel.astype(bool)


def _queries(queries, c_ins):
    from paper_2604_10982_b200.panoptic import pack_queries
    return pack_queries(queries, c_ins)


def assign_labels(surfels13, f_ins, queries):
    """assign_labels (panoptic.cpp:36-91) by the reference: (dist (N, Q) per-surfel rows, argmax (N,))."""
    s = np.ascontiguousarray(np.asarray(surfels13, dtype=np.float64).reshape(-1, 13))
    n = s.shape[0]
    f = np.ascontiguousarray(np.asarray(f_ins, dtype=np.float64).reshape(n, -1))
    feat, mean, cov, alive, _ = _queries(queries, f.shape[1])
    q = len(queries)
    dist = np.zeros((n, q))
    arg = np.zeros(n, np.int32)
    if load().ref_assign_labels(_p(s), n, _p(f), f.shape[1], q, _p(feat), _p(mean), _p(cov), _p(alive), _p(dist),
                                _p(arg)) != 0:
        raise ValueError("assign_labels failed")
    return dist, arg


class RefPanopticScene:
    """A panoptic psimap::SceneMap (f_sem, f_ins, instance queries) held by the reference library, so
    that render_panoptic (metrics.cpp:339-369: assign_labels, render, epilogue) can be timed alone."""

    def __init__(self, scene):
        self.lib = load()
        s = np.ascontiguousarray(scene.surfels)
        f = np.ascontiguousarray(scene.f_sem)
        fi = np.ascontiguousarray(scene.f_ins)
        feat, mean, cov, alive, cls = _queries(scene.queries, fi.shape[1])
        self._keep = (s, f, fi, feat, mean, cov, alive, cls)
        self.h = self.lib.ref_panoptic_scene_create(_p(s), s.shape[0], _p(f), f.shape[1], _p(fi), fi.shape[1],
                                                    len(scene.queries), _p(feat), _p(mean), _p(cov), _p(alive),
                                                    _p(cls))

    def render(self, cam_c, cfg_c, out=None) -> None:
        ids, classes, sem = (None, None, None) if out is None else out
        if self.lib.ref_render_panoptic_h(self.h, C.byref(cam_c), C.byref(cfg_c), _p(ids), _p(classes), _p(sem)) != 0:
            raise ValueError("render_panoptic failed")

    def close(self):
        if self.h:
            self.lib.ref_panoptic_scene_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def render_panoptic(scene, cam, cfg) -> dict:
    """render_panoptic (metrics.cpp:339-369) by the reference over scene.surfels / f_sem / f_ins / queries."""
    s = scene.surfels
    n = s.shape[0]
    f = np.ascontiguousarray(scene.f_sem)
    fi = np.ascontiguousarray(scene.f_ins)
    feat, mean, cov, alive, cls = _queries(scene.queries, fi.shape[1])
    w, h = cam.width, cam.height
    out = {k: np.zeros((h, w, 1), np.int32) for k in ("ids", "classes", "sem_classes")}
    if load().ref_render_panoptic(_p(s), n, _p(f), f.shape[1], _p(fi), fi.shape[1], len(scene.queries), _p(feat),
                                  _p(mean), _p(cov), _p(alive), _p(cls), C.byref(cam.to_c()), C.byref(cfg.to_c()),
                                  _p(out["ids"]), _p(out["classes"]), _p(out["sem_classes"])) != 0:
        raise ValueError("render_panoptic failed")
    return out
