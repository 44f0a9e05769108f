"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/psm.h declares,
its host-only entry points work without a GPU, and the render path refuses to run without one
(no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np

from paper_2604_10982_b200 import _abi as A
from paper_2604_10982_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "psm.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(psm_\w+)\s*\(", text, re.M)))


def test_header_matches_python_symbol_list():
    assert _declared_symbols() == sorted(A.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_lib.LIB_PATH)
    for name in _declared_symbols():
        assert hasattr(lib, name), name


def test_no_oracle_in_product_library():
    """The product library must not contain the oracle (no CPU render path)."""
    lib = C.CDLL(_lib.LIB_PATH)
    for name in ("oracle_render", "oracle_bin", "oracle_project_surfel"):
        assert not hasattr(lib, name)


def test_default_config_matches_reference():
    lib = _lib.load()
    c = A.psm_raster_config()
    lib.psm_default_config(C.byref(c))
    assert (c.tile_size, c.chi2, c.alpha_min, c.t_min, c.support_cutoff, c.binning, c.blending, c.top_k,
            c.render_depth_normal) == (16, 9.0, 1.0 / 255.0, 1e-4, 1, A.BIN_AABB, A.BLEND_FULL, 16, 1)


def test_render_refuses_without_gpu():
    import torch
    if torch.cuda.is_available():
        return
    lib = _lib.load()
    ctx = C.c_void_p()
    assert lib.psm_create(0, None, C.byref(ctx)) == A.PSM_ECUDA


def test_camera_factories_validate():
    import pytest
    from paper_2604_10982_b200 import Camera
    with pytest.raises(ValueError):
        Camera.make(np.eye(3), np.zeros(3), 0.0, 1.0, 0, 0, 4, 4, 0.1, 10)
    with pytest.raises(ValueError):
        Camera.look_at((0, 0, 0), (0, 0, 0), (0, -1, 0), 1, 1, 4, 4, 0.1, 10)
    cam = Camera.look_at((0, 0, 0), (0, 0, 20), (0, -1, 0), 204.8, 204.8, 256, 192, 0.1, 200.0)
    # core_types.cpp:40-60: image +y points down, cx = W/2
    assert cam.cx == 128.0 and cam.cy == 96.0
    # right = fwd x up = +x, down = fwd x right = +y: the street camera is the identity pose
    assert np.array_equal(cam.r_cw, np.eye(3)) and np.array_equal(cam.t_cw, np.zeros(3))


def test_street_scene_shape_and_determinism():
    from paper_2604_10982_b200 import StreetSpec, make_street_scene
    a, la, cam = make_street_scene(StreetSpec(n_surfels=2000, c_sem=4, n_instances=16))
    b, lb, _ = make_street_scene(StreetSpec(n_surfels=2000, c_sem=4, n_instances=16))
    assert a.surfels.shape[1] == 13 and a.f_sem.shape == (len(a), 4) and la.shape == (len(a), 16)
    assert np.array_equal(a.surfels, b.surfels) and np.array_equal(a.f_sem, b.f_sem)
    q = a.surfels[:, 3:7]
    assert np.allclose(np.linalg.norm(q, axis=1), 1.0, atol=1e-12)
    assert np.all(a.surfels[:, 8] * 5.0 <= a.surfels[:, 7] + 1e-12)  # aspect >= min_aspect
    assert np.all((la == 0.92) | np.isclose(la, 0.08 / 15))
    assert cam.width == 256 and cam.height == 192 and cam.fx == 0.8 * 256
