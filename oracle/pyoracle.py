"""ctypes wrapper of the CPU oracle (oracle/oracle.cpp). TEST INFRASTRUCTURE ONLY:
imported by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs, never
by the product package.

Parity pin: see the header of oracle/oracle.cpp (restatement of
proj/src/raster.cpp pinned by the reference's known-answer tests, ported in
tests/test_oracle_kat.py; bit-level agreement with an Eigen build of the
reference is unpinned because the reference cannot be built here).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

from paper_2604_10982_b200 import _abi as A

HERE = os.path.dirname(os.path.abspath(__file__))
_libs = {}


class oracle_stats(C.Structure):
    _fields_ = [("candidates_tested", C.c_uint64), ("support_pass", C.c_uint64), ("contributors", C.c_uint64),
                ("t_project_ms", C.c_double), ("t_bin_ms", C.c_double), ("t_blend_ms", C.c_double),
                ("t_total_ms", C.c_double)]


class oracle_projected(C.Structure):
    _fields_ = [("status", C.c_int32), ("center", C.c_double * 2), ("sigma", C.c_double * 4),
                ("sort_depth", C.c_double), ("h", C.c_double * 9), ("h_inv", C.c_double * 9),
                ("finv", C.c_double * 4), ("normal_vis", C.c_double * 3)]


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def load(libm: bool = False):
    """libm=False: psm_exp (bit-parity oracle); libm=True: glibc exp exactly as raster.cpp:390."""
    key = "libm" if libm else "parity"
    if key in _libs:
        return _libs[key]
    path = os.path.join(HERE, "liboracle_libm.so" if libm else "liboracle.so")
    if not os.path.exists(path):
        build()
    lib = C.CDLL(path)
    vp, P = C.c_void_p, C.POINTER
    lib.oracle_render.restype = C.c_int
    lib.oracle_render.argtypes = [vp, C.c_int64, vp, C.c_int32, vp, C.c_int32, P(A.psm_camera),
                                  P(A.psm_raster_config)] + [vp] * 8 + [P(A.psm_counters), P(A.psm_debug),
                                                                         P(oracle_stats)]
    lib.oracle_project_surfel.restype = C.c_int
    lib.oracle_project_surfel.argtypes = [vp, P(A.psm_camera), C.c_double, P(oracle_projected)]
    lib.oracle_evaluate_alpha.restype = C.c_double
    lib.oracle_evaluate_alpha.argtypes = [vp, P(A.psm_camera), C.c_double, C.c_double, P(A.psm_raster_config),
                                          P(C.c_double), P(C.c_double), P(C.c_double), P(C.c_int32)]
    lib.oracle_bin.restype = C.c_int
    lib.oracle_bin.argtypes = [vp, C.c_int64, P(A.psm_camera), P(A.psm_raster_config), C.c_int32, C.c_double,
                               vp, vp, C.c_int64, vp, P(A.psm_counters)]
    lib.oracle_project_surfel_backward.restype = C.c_int
    lib.oracle_project_surfel_backward.argtypes = [vp, P(A.psm_camera), C.c_double, vp, vp, vp, vp]
    lib.oracle_topk_select.restype = None
    lib.oracle_topk_select.argtypes = [vp, vp, C.c_int32, C.c_int32, vp]
    _libs[key] = lib
    return lib


def _p(a: Optional[np.ndarray]):
    return None if a is None or a.size == 0 else a.ctypes.data_as(C.c_void_p)


def project_surfel(s13, cam, chi2: float = 9.0) -> dict:
    s = np.ascontiguousarray(np.asarray(s13, dtype=np.float64).reshape(13))
    out = oracle_projected()
    c = cam.to_c()
    st = load().oracle_project_surfel(_p(s), C.byref(c), chi2, C.byref(out))
    if st < 0:
        raise ValueError("degenerate quaternion")
    if st == 0:
        return None
    return {
        "center": np.array(list(out.center)),
        "sigma": np.array(list(out.sigma)).reshape(2, 2).T,
        "sort_depth": out.sort_depth,
        "h": np.array(list(out.h)).reshape(3, 3).T,
        "h_inv": np.array(list(out.h_inv)).reshape(3, 3).T,
        "footprint_inv": np.array(list(out.finv)).reshape(2, 2).T,
        "normal_vis": np.array(list(out.normal_vis)),
    }


def project_surfel_backward(s13, cam, g_hinv, chi2: float = 9.0) -> Optional[dict]:
    """project_surfel_backward (raster.cpp:179-203) through psm_geom_backward: d L / d (centre,
    quaternion, scales) from d L / d H^-1 (3x3). None when the surfel does not project."""
    s = np.ascontiguousarray(np.asarray(s13, dtype=np.float64).reshape(13))
    g = np.ascontiguousarray(np.asarray(g_hinv, dtype=np.float64).reshape(3, 3))
    dc, dq, ds = np.zeros(3), np.zeros(4), np.zeros(2)
    st = load().oracle_project_surfel_backward(_p(s), C.byref(cam.to_c()), chi2, _p(g), _p(dc), _p(dq), _p(ds))
    if st < 0:
        raise ValueError("degenerate quaternion")
    return None if st == 0 else {"center": dc, "rotation": dq, "scales": ds}


def evaluate_alpha(s13, cam, px: float, py: float, cfg) -> dict:
    s = np.ascontiguousarray(np.asarray(s13, dtype=np.float64).reshape(13))
    u, v, w2, inside = C.c_double(), C.c_double(), C.c_double(), C.c_int32()
    c, k = cam.to_c(), cfg.to_c()
    a = load().oracle_evaluate_alpha(_p(s), C.byref(c), px, py, C.byref(k), C.byref(u), C.byref(v), C.byref(w2),
                                     C.byref(inside))
    return {"alpha": a, "u": u.value, "v": v.value, "w2": w2.value, "inside": bool(inside.value)}


def bin_surfels(surfels13, cam, cfg, binning: int, chi2: Optional[float] = None) -> dict:
    """Projects + bins (bin_circle / bin_aabb / ellipse). Returns per-tile lists of source ids."""
    s = np.ascontiguousarray(np.asarray(surfels13, dtype=np.float64).reshape(-1, 13))
    n = s.shape[0]
    c, k = cam.to_c(), cfg.to_c()
    tiles = ((cam.width + cfg.tile_size - 1) // cfg.tile_size) * ((cam.height + cfg.tile_size - 1) // cfg.tile_size)
    counts = np.zeros(tiles, dtype=np.int32)
    per = np.zeros(max(n, 1), dtype=np.int32)
    cnt = A.psm_counters()
    lib = load()
    chi = cfg.chi2 if chi2 is None else chi2
    st = lib.oracle_bin(_p(s), n, C.byref(c), C.byref(k), binning, chi, _p(counts), None, 0, _p(per), C.byref(cnt))
    if st != 0:
        raise ValueError("degenerate quaternion")
    total = int(counts.sum())
    lists = np.zeros(max(total, 1), dtype=np.int32)
    lib.oracle_bin(_p(s), n, C.byref(c), C.byref(k), binning, chi, None, _p(lists), total, None, None)
    offs = np.concatenate([[0], np.cumsum(counts)])
    return {"tiles": [lists[offs[t]:offs[t + 1]].copy() for t in range(tiles)], "rn_total": int(cnt.rn_total),
            "rn_per_tile": float(cnt.rn_per_tile), "per_surfel": per[:n].copy(), "n_proj": int(cnt.n_proj)}


def make_street_scene(spec, with_labels: bool = False, with_f_ins: bool = False):
    """make_street_scene (synthetic.cpp:236-312, + scale_mult) on the oracle: (surfels13 (N,13),
    f_sem (N,C), labels (N,n_instances) or None, psm_camera[, f_ins (N,8)]). Loads no product code."""
    lib = load()
    fn = lib.oracle_make_street_scene
    fn.restype = C.c_int
    fn.argtypes = [C.POINTER(A.psm_street_spec), C.POINTER(C.c_int64), C.c_void_p, C.c_void_p, C.c_void_p,
                   C.c_void_p, C.POINTER(A.psm_camera)]
    cs = spec.to_c()
    n = C.c_int64()
    cam = A.psm_camera()
    if fn(C.byref(cs), C.byref(n), None, None, None, None, C.byref(cam)) != 0:
        raise ValueError("make_street_scene failed")
    s = np.empty((n.value, 13))
    f = np.empty((n.value, spec.c_sem))
    lab = np.empty((n.value, spec.n_instances)) if with_labels else None
    fi = np.empty((n.value, 8)) if with_f_ins else None
    fn(C.byref(cs), C.byref(n), _p(s), _p(f), _p(lab), _p(fi), C.byref(cam))
    return (s, f, lab, cam, fi) if with_f_ins else (s, f, lab, cam)


def psm_exp(x) -> np.ndarray:
    xs = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    out = np.empty_like(xs)
    fn = load().oracle_psm_exp
    fn.restype = None
    fn.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
    fn(_p(xs), xs.size, _p(out))
    return out


def libm_exp(x) -> np.ndarray:
    """glibc exp (the reference's libm), called from C++ std::exp."""
    xs = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    out = np.empty_like(xs)
    fn = load().oracle_libm_exp
    fn.restype = None
    fn.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
    fn(_p(xs), xs.size, _p(out))
    return out


def host_uses_fma_exp() -> bool:
    """glibc's ifunc picks the FMA build of exp on CPUs with FMA and AVX2."""
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:
        return False
    return " fma" in flags and " avx2" in flags


def topk_select(weights, proj, k: int) -> np.ndarray:
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
    p = np.ascontiguousarray(np.asarray(proj, dtype=np.int32))
    sel = np.zeros(len(w), dtype=np.int8)
    load().oracle_topk_select(_p(w), _p(p), len(w), k, _p(sel))
    return sel.astype(bool)


def render(scene, labels, cam, cfg, debug: bool = False, libm: bool = False, planes=True) -> dict:
    """render_into (raster.cpp:273-511) on the CPU oracle. Returns fp64 planes (H, W, C),
    counters, optional debug exports (sorted keys, ranges, depth order, Top-K ids) and stats."""
    lib = load(libm)
    s = scene.surfels
    n = s.shape[0]
    w, h = cam.width, cam.height
    c_sem = scene.c_sem()
    lab = None if labels is None else np.ascontiguousarray(np.asarray(labels, dtype=np.float64))
    n_q = 0 if lab is None else lab.shape[1]
    npx = w * h
    out = {
        "color": np.zeros((h, w, 3)), "depth": np.zeros((h, w, 2)), "normal": np.zeros((h, w, 3)),
        "sem_feat": np.zeros((h, w, c_sem)), "ins_dist": np.zeros((h, w, n_q)),
        "ins_argmax": np.zeros((h, w, 1), dtype=np.int32), "alpha_acc": np.zeros((h, w, 1)),
        "blend_count": np.zeros((h, w, 1), dtype=np.int32),
    } if planes else {"color": np.zeros((h, w, 3)), "alpha_acc": np.zeros((h, w, 1)),
                      "blend_count": np.zeros((h, w, 1), dtype=np.int32),
                      "ins_argmax": np.zeros((h, w, 1), dtype=np.int32)}
    cnt = A.psm_counters()
    st_ = oracle_stats()
    dbg = None
    k_sel = max(cfg.top_k, 1)
    if debug:
        cap = 1 << 26
        # size the key buffers from a counting pass
        c0 = A.psm_counters()
        lib.oracle_render(_p(s), n, _p(scene.f_sem), c_sem, _p(lab), n_q, C.byref(cam.to_c()), C.byref(cfg.to_c()),
                          *[None] * 8, C.byref(c0), None, None)
        cap = max(int(c0.rn_total), 1)
        out["tile_keys"] = np.zeros(cap, dtype=np.uint64)
        out["tile_vals"] = np.zeros(cap, dtype=np.int32)
        tiles = ((w + cfg.tile_size - 1) // cfg.tile_size) * ((h + cfg.tile_size - 1) // cfg.tile_size)
        out["tile_ranges"] = np.zeros((tiles, 2), dtype=np.int32)
        out["depth_order"] = np.zeros(max(int(c0.n_proj), 1), dtype=np.int32)
        out["topk_src"] = np.full((h, w, k_sel), -1, dtype=np.int32)
        dbg = A.psm_debug(_p(out["tile_keys"]), _p(out["tile_vals"]), cap, _p(out["tile_ranges"]),
                          _p(out["depth_order"]), int(c0.n_proj), _p(out["topk_src"]))
    status = lib.oracle_render(_p(s), n, _p(scene.f_sem), c_sem, _p(lab), n_q, C.byref(cam.to_c()),
                               C.byref(cfg.to_c()), _p(out.get("color")), _p(out.get("depth")),
                               _p(out.get("normal")), _p(out.get("sem_feat")), _p(out.get("ins_dist")),
                               _p(out.get("ins_argmax")), _p(out.get("alpha_acc")), _p(out.get("blend_count")),
                               C.byref(cnt), C.byref(dbg) if dbg is not None else None, C.byref(st_))
    if status == A.PSM_EINVAL:
        raise ValueError("degenerate quaternion")
    if status != 0:
        raise RuntimeError(f"oracle status {status}")
    out["counters"] = cnt.as_dict()
    out["stats"] = {k: getattr(st_, k) for k, _ in st_._fields_}
    if debug:
        out["depth_order"] = out["depth_order"][: int(cnt.n_proj)]
        out["tile_keys"] = out["tile_keys"][: int(cnt.rn_total)]
        out["tile_vals"] = out["tile_vals"][: int(cnt.rn_total)]
    return out


class oracle_cache(C.Structure):
    _fields_ = [("offsets", C.c_void_p), ("src", C.c_void_p), ("alpha", C.c_void_p), ("cap", C.c_int64)]


def render_cache(scene, labels, cam, cfg) -> dict:
    """render(..., &cache): planes (color, sem_feat, ins_argmax, blend_count) plus the per-pixel
    contributor lists of RenderCache::pixels (raster.cpp:399-403) as CSR (offsets, source, alpha)."""
    lib = load()
    fn = lib.oracle_render_cache
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.POINTER(A.psm_camera),
                   C.POINTER(A.psm_raster_config), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                   C.POINTER(oracle_cache)]
    s = scene.surfels
    w, h = cam.width, cam.height
    c_sem = scene.c_sem()
    lab = None if labels is None else np.ascontiguousarray(np.asarray(labels, dtype=np.float64))
    n_q = 0 if lab is None else lab.shape[1]
    color = np.zeros((h, w, 3))
    sem = np.zeros((h, w, c_sem))
    arg = np.zeros((h, w, 1), dtype=np.int32)
    cnt = np.zeros((h, w, 1), dtype=np.int32)
    offs = np.zeros(w * h + 1, dtype=np.int64)
    cache = oracle_cache(_p(offs), None, None, 0)
    st = fn(_p(s), s.shape[0], _p(scene.f_sem), c_sem, _p(lab), n_q, C.byref(cam.to_c()), C.byref(cfg.to_c()),
            _p(color), _p(sem), _p(arg), _p(cnt), C.byref(cache))
    if st != 0:
        raise ValueError("oracle render failed")
    total = int(offs[-1])
    src = np.zeros(max(total, 1), dtype=np.int32)
    alpha = np.zeros(max(total, 1))
    cache = oracle_cache(_p(offs), _p(src), _p(alpha), total)
    fn(_p(s), s.shape[0], _p(scene.f_sem), c_sem, _p(lab), n_q, C.byref(cam.to_c()), C.byref(cfg.to_c()),
       _p(color), _p(sem), _p(arg), _p(cnt), C.byref(cache))
    return {"color": color, "sem_feat": sem, "ins_argmax": arg, "blend_count": cnt, "offsets": offs,
            "src": src[:total], "alpha": alpha[:total]}


def assign_labels(surfels13, f_ins, queries, threads: int = 0):
    """assign_labels (panoptic.cpp:36-91) on the oracle: (dist (N, Q) per-surfel rows, argmax (N,))."""
    from paper_2604_10982_b200.panoptic import pack_queries
    lib = load()
    fn = lib.oracle_assign_labels
    fn.restype = None
    vp = C.c_void_p
    fn.argtypes = [vp, C.c_int64, vp, C.c_int32, C.c_int32, vp, vp, vp, vp, vp, vp, C.c_int32]
    s = np.ascontiguousarray(np.asarray(surfels13, dtype=np.float64).reshape(-1, 13))
    n = s.shape[0]
    f = np.ascontiguousarray(np.asarray(f_ins, dtype=np.float64).reshape(n, -1))
    c_ins = f.shape[1]
    feat, mean, cov, alive, _ = pack_queries(queries, c_ins)
    q = len(queries)
    dist = np.zeros((n, q))
    arg = np.full(n, -1, np.int32)
    if n:
        fn(_p(s), n, _p(f), c_ins, q, _p(feat), _p(mean), _p(cov), _p(alive), _p(dist), _p(arg), threads)
    return dist, arg


def render_panoptic(scene, f_ins, queries, cam, cfg) -> dict:
    """render_panoptic (metrics.cpp:339-369): assign_labels, render with the label
    distribution, then the per-pixel epilogue over the fp64 planes."""
    from paper_2604_10982_b200.panoptic import panoptic_epilogue
    dist, arg = assign_labels(scene.surfels, f_ins, queries)
    labels = dist if len(queries) else None
    out = render(scene, labels, cam, cfg)
    pr = panoptic_epilogue(out["alpha_acc"], out["ins_argmax"], out["sem_feat"], [q.class_id for q in queries])
    out.update(ids=pr.ids, classes=pr.classes, sem_classes=pr.sem_classes, dist=dist, label_argmax=arg)
    return out


def render_backward(scene, labels, cam, cfg, g_color=None, g_sem=None, g_ins=None) -> dict:
    """Blending backward + project_surfel_backward (pipeline.cpp:347-486) on the oracle: gradients of
    L = <g_color, colour> + <g_sem, sem_feat> + <g_ins, ins_dist> w.r.t. every surfel parameter."""
    lib = load()
    fn = lib.oracle_render_backward
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.POINTER(A.psm_camera),
                   C.POINTER(A.psm_raster_config), C.POINTER(A.psm_plane_grads), C.POINTER(A.psm_scene_grads)]
    s = scene.surfels
    n = s.shape[0]
    c_sem = scene.c_sem()
    lab = None if labels is None else np.ascontiguousarray(np.asarray(labels, dtype=np.float64))
    n_q = 0 if lab is None else lab.shape[1]
    gp = [None if a is None else np.ascontiguousarray(a, dtype=np.float64) for a in (g_color, g_sem, g_ins)]
    out = {"opacity": np.zeros(n), "color": np.zeros((n, 3)), "f_sem": np.zeros((n, c_sem)),
           "labels": np.zeros((n, n_q)), "center": np.zeros((n, 3)), "rotation": np.zeros((n, 4)),
           "scales": np.zeros((n, 2))}
    pg = A.psm_plane_grads(*[_p(a) for a in gp])
    sg = A.psm_scene_grads(*[_p(out[k]) for k in ("opacity", "color", "f_sem", "labels", "center", "rotation",
                                                    "scales")])
    st = fn(_p(s), n, _p(scene.f_sem), c_sem, _p(lab), n_q, C.byref(cam.to_c()), C.byref(cfg.to_c()), C.byref(pg),
            C.byref(sg))
    if st != 0:
        raise ValueError("oracle backward failed")
    return out
