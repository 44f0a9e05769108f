"""Loader for the in-tree CUDA library `paper_2604_10982_b200/libpsm.so`.

There is no CPU fallback: if the library is missing, `load()` raises. Build it
with `python -c "import __graft_entry__ as g; g.build()"` (or `make -C
paper_2604_10982_b200/csrc`).
"""
import ctypes as C
import os

from . import _abi as A

# PSM_LIB_PATH selects another build of the same library (A/B kernel variants under scratch/)
LIB_PATH = os.environ.get("PSM_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpsm.so")
_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"CUDA extension not built: {LIB_PATH} missing (run __graft_entry__.build())")
    lib = C.CDLL(LIB_PATH)
    P = C.POINTER
    vp = C.c_void_p
    sig = {
        "psm_default_config": (None, [P(A.psm_raster_config)]),
        "psm_create": (C.c_int, [C.c_int, vp, P(vp)]),
        "psm_destroy": (C.c_int, [vp]),
        "psm_last_error": (C.c_char_p, [vp]),
        "psm_set_profiling": (C.c_int, [vp, C.c_int]),
        "psm_get_stage_times": (C.c_int, [vp, P(A.psm_stage_times)]),
        "psm_sync": (C.c_int, [vp]),
        "psm_scene_upload": (C.c_int, [vp, vp, C.c_int64, vp, C.c_int32, vp, C.c_int32, P(vp)]),
        "psm_scene_free": (C.c_int, [vp, vp]),
        "psm_scene_info": (C.c_int, [vp, P(C.c_int64), P(C.c_int32), P(C.c_int32)]),
        "psm_render": (C.c_int, [vp, vp, P(A.psm_camera), P(A.psm_raster_config), P(A.psm_targets),
                                 P(A.psm_counters)]),
        "psm_render_debug": (C.c_int, [vp, vp, P(A.psm_camera), P(A.psm_raster_config), P(A.psm_targets),
                                       P(A.psm_counters), P(A.psm_debug)]),
        "psm_scene_create": (C.c_int, [vp, P(A.psm_scene_desc), P(vp)]),
        "psm_assign_labels": (C.c_int, [vp, vp, P(A.psm_queries), vp, vp]),
        "psm_render_panoptic": (C.c_int, [vp, vp, P(A.psm_camera), P(A.psm_raster_config), vp, C.c_int32,
                                          P(A.psm_panoptic_targets), P(A.psm_counters)]),
        "psm_make_street_scene_ins": (C.c_int, [P(A.psm_street_spec), P(C.c_int64), vp]),
        "psm_render_backward": (C.c_int, [vp, vp, P(A.psm_camera), P(A.psm_raster_config), P(A.psm_plane_grads),
                                          P(A.psm_scene_grads)]),
        "psm_render_batch": (C.c_int, [vp, vp, P(A.psm_camera), C.c_int32, P(A.psm_raster_config),
                                       P(A.psm_targets), P(A.psm_counters)]),
        "psm_last_counters": (C.c_int, [vp, P(A.psm_counters)]),
        "psm_project_surfels": (C.c_int, [vp, vp, C.c_int64, P(A.psm_camera), P(A.psm_raster_config), vp, vp,
                                          P(C.c_int64)]),
        "psm_bin_projected": (C.c_int, [vp, vp, C.c_int64, P(A.psm_camera), P(A.psm_raster_config), C.c_int32,
                                        C.c_double, vp, vp, C.c_int64, P(A.psm_counters)]),
        "psm_sample_alpha": (C.c_int, [vp, vp, vp, C.c_int64, vp, vp, vp, C.c_int64, P(A.psm_camera),
                                       P(A.psm_raster_config), vp]),
        "psm_topk_select": (C.c_int, [vp, vp, vp, vp, C.c_int32, C.c_int32, vp]),
        "psm_render_cache": (C.c_int, [vp, vp, P(A.psm_camera), P(A.psm_raster_config), P(A.psm_targets),
                                       P(A.psm_counters), P(A.psm_render_cache_out)]),
        "psm_make_street_scene": (C.c_int, [P(A.psm_street_spec), P(C.c_int64), vp, vp, vp, P(A.psm_camera)]),
        "psm_camera_look_at": (C.c_int, [P(C.c_double * 3), P(C.c_double * 3), P(C.c_double * 3), C.c_double,
                                         C.c_double, C.c_int32, C.c_int32, C.c_double, C.c_double,
                                         P(A.psm_camera)]),
        "psm_camera_make": (C.c_int, [P(C.c_double * 9), P(C.c_double * 3), C.c_double, C.c_double, C.c_double,
                                      C.c_double, C.c_int32, C.c_int32, C.c_double, C.c_double, P(A.psm_camera)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
