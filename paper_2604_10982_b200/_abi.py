"""ctypes mirrors of the structs in include/psm.h (no library is loaded here).

Kept separate from `_lib` so the test-side oracle wrapper can share the exact
struct layouts without loading the CUDA library.
"""
import ctypes as C

PSM_OK = 0
PSM_EINVAL = 1
PSM_ENOMEM = 2
PSM_ECUDA = 3
PSM_EUNSUPPORTED = 4

BIN_CIRCLE, BIN_AABB, BIN_ELLIPSE = 0, 1, 2
BLEND_FULL, BLEND_TOPK = 0, 1


class psm_camera(C.Structure):
    _fields_ = [("r_cw", C.c_double * 9), ("t_cw", C.c_double * 3), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("width", C.c_int32), ("height", C.c_int32),
                ("near_clip", C.c_double), ("far_clip", C.c_double)]


class psm_raster_config(C.Structure):
    _fields_ = [("tile_size", C.c_int32), ("chi2", C.c_double), ("alpha_min", C.c_double), ("t_min", C.c_double),
                ("support_cutoff", C.c_int32), ("binning", C.c_int32), ("blending", C.c_int32), ("top_k", C.c_int32),
                ("background", C.c_double * 3), ("render_depth_normal", C.c_int32), ("threads", C.c_int32)]


class psm_targets(C.Structure):
    _fields_ = [("color", C.c_void_p), ("depth", C.c_void_p), ("normal", C.c_void_p), ("sem_feat", C.c_void_p),
                ("ins_dist", C.c_void_p), ("ins_argmax", C.c_void_p), ("alpha_acc", C.c_void_p),
                ("blend_count", C.c_void_p), ("on_device", C.c_int32)]


class psm_counters(C.Structure):
    _fields_ = [("rn_total", C.c_uint64), ("rn_per_tile", C.c_double), ("blended_total", C.c_uint64),
                ("n_proj", C.c_int64), ("tiles_x", C.c_int32), ("tiles_y", C.c_int32), ("nonempty_tiles", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class psm_debug(C.Structure):
    _fields_ = [("tile_keys", C.c_void_p), ("tile_vals", C.c_void_p), ("cap_keys", C.c_int64),
                ("tile_ranges", C.c_void_p), ("depth_order", C.c_void_p), ("cap_proj", C.c_int64),
                ("topk_src", C.c_void_p)]


class psm_stage_times(C.Structure):
    _fields_ = [("preprocess", C.c_float), ("tile_scan", C.c_float), ("emit", C.c_float), ("tile_sort", C.c_float),
                ("blend", C.c_float), ("total", C.c_float)]

    def as_dict(self):
        return {k: float(getattr(self, k)) for k, _ in self._fields_}


class psm_street_spec(C.Structure):
    _fields_ = [("n_surfels", C.c_int32), ("seed", C.c_uint64), ("min_aspect", C.c_double), ("image_w", C.c_int32),
                ("image_h", C.c_int32), ("c_sem", C.c_int32), ("n_instances", C.c_int32), ("scale_mult", C.c_double)]


PSM_SCENE_EXACT_FEATURES = 1


class psm_scene_desc(C.Structure):
    _fields_ = [("surfels13", C.c_void_p), ("n", C.c_int64), ("f_sem", C.c_void_p), ("c_sem", C.c_int32),
                ("labels", C.c_void_p), ("n_q", C.c_int32), ("f_ins", C.c_void_p), ("c_ins", C.c_int32),
                ("flags", C.c_int32)]


class psm_queries(C.Structure):
    _fields_ = [("n", C.c_int32), ("c_ins", C.c_int32), ("feature", C.c_void_p), ("mean", C.c_void_p),
                ("cov", C.c_void_p), ("alive", C.c_void_p), ("class_id", C.c_void_p)]


class psm_panoptic_targets(C.Structure):
    _fields_ = [("ids", C.c_void_p), ("classes", C.c_void_p), ("sem_classes", C.c_void_p), ("on_device", C.c_int32)]


class psm_plane_grads(C.Structure):
    _fields_ = [("color", C.c_void_p), ("sem_feat", C.c_void_p), ("ins_dist", C.c_void_p)]


class psm_scene_grads(C.Structure):
    _fields_ = [("opacity", C.c_void_p), ("color", C.c_void_p), ("f_sem", C.c_void_p), ("labels", C.c_void_p),
                ("center", C.c_void_p), ("rotation", C.c_void_p), ("scales", C.c_void_p)]


class psm_projected(C.Structure):  # ProjectedSurfel (raster.hpp:21-30); matrices column-major
    _fields_ = [("source", C.c_int32), ("pad", C.c_int32), ("screen_center", C.c_double * 2),
                ("sigma", C.c_double * 4), ("sort_depth", C.c_double), ("h", C.c_double * 9),
                ("h_inv", C.c_double * 9), ("footprint_inv", C.c_double * 4), ("normal_vis", C.c_double * 3)]


class psm_alpha_sample(C.Structure):  # AlphaSample (raster.hpp:103-108) + evaluate_alpha's alpha
    _fields_ = [("alpha", C.c_double), ("u", C.c_double), ("v", C.c_double), ("w2", C.c_double),
                ("inside", C.c_int32), ("pad", C.c_int32)]


class psm_contribution(C.Structure):  # PixelContribution (raster.hpp:69-74)
    _fields_ = [("proj", C.c_int32), ("pad", C.c_int32), ("alpha", C.c_double), ("u", C.c_double),
                ("v", C.c_double)]


class psm_render_cache_out(C.Structure):
    _fields_ = [("projected", C.c_void_p), ("projected_cap", C.c_int64), ("n_projected", C.c_int64),
                ("tile_counts", C.c_void_p), ("tile_lists", C.c_void_p), ("tile_lists_cap", C.c_int64),
                ("n_tile_entries", C.c_int64), ("pixel_offsets", C.c_void_p), ("contribs", C.c_void_p),
                ("contribs_cap", C.c_int64), ("n_contribs", C.c_int64)]


# Every symbol include/psm.h declares (checked by tests/test_capi_symbols.py).
EXPORTED_SYMBOLS = (
    "psm_default_config", "psm_create", "psm_destroy", "psm_last_error", "psm_set_profiling", "psm_get_stage_times",
    "psm_sync", "psm_scene_upload", "psm_scene_free", "psm_scene_info", "psm_render", "psm_render_debug",
    "psm_render_batch", "psm_last_counters", "psm_make_street_scene", "psm_camera_look_at", "psm_camera_make",
    "psm_scene_create", "psm_assign_labels", "psm_render_panoptic", "psm_make_street_scene_ins",
    "psm_render_backward", "psm_project_surfels", "psm_bin_projected", "psm_sample_alpha", "psm_topk_select",
    "psm_render_cache",
)
