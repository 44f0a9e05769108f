"""GPU render backward against the oracle backward (which the
finite-difference suite in tests/test_backward_oracle.py pins, and tests/test_ref_pin.py pins bit
for bit to the reference's own pipeline_backward): every gradient within fp64 summation-order noise
(the GPU sums per-surfel contributions with atomics)."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2604_10982_b200 import (Binning, Blending, RasterConfig, Renderer, SceneMap, StreetSpec,
                                   make_street_scene)
from tests.helpers import front_camera
from tests.test_backward_oracle import scene_case

pytestmark = pytest.mark.gpu
KEYS = ("opacity", "color", "f_sem", "labels", "center", "rotation", "scales")


@pytest.fixture(scope="module")
def rend():
    r = Renderer(0)
    yield r
    r.close()


def assert_grads_close(g, o):
    for k in KEYS:
        a, b = g[k], o[k]
        assert a.shape == b.shape, k
        if b.size:
            scale = max(np.max(np.abs(b)), 1e-300)
            err = np.max(np.abs(a - b))
            assert err <= 1e-9 * scale, (k, err, scale)


@pytest.mark.parametrize("blending,k", [(Blending.Full, 16), (Blending.TopK, 2)])
def test_gpu_backward_small(rend, blending, k):
    scene, lab = scene_case(5)
    cam = front_camera(32, 32, 60.0)
    cfg = RasterConfig(blending=blending, top_k=k)
    rng = np.random.default_rng(9)
    gc, gs, gi = rng.normal(size=(32, 32, 3)), rng.normal(size=(32, 32, 3)), rng.normal(size=(32, 32, 2))
    assert_grads_close(rend.render_backward(scene, lab, cam, cfg, gc, gs, gi),
                       O.render_backward(scene, lab, cam, cfg, gc, gs, gi))


@pytest.mark.parametrize("blending,binning", [(Blending.TopK, Binning.Ellipse), (Blending.Full, Binning.Aabb)])
def test_gpu_backward_street(rend, blending, binning):
    sc, labels, cam = make_street_scene(StreetSpec(n_surfels=12000, image_w=256, image_h=192, c_sem=8,
                                                   n_instances=6, seed=7))
    cfg = RasterConfig(binning=binning, blending=blending, top_k=16)
    rng = np.random.default_rng(3)
    gc = rng.normal(size=(192, 256, 3))
    gs = rng.normal(size=(192, 256, 8))
    gi = rng.normal(size=(192, 256, labels.shape[1]))
    g = rend.render_backward(sc, labels, cam, cfg, gc, gs, gi)
    o = O.render_backward(sc, labels, cam, RasterConfig(binning=Binning.Aabb, blending=blending, top_k=16), gc, gs, gi)
    assert_grads_close(g, o)
    assert np.count_nonzero(g["center"]) > 0.05 * g["center"].size  # visible (unoccluded) surfels


def test_gpu_backward_zero_upstream(rend):
    scene, lab = scene_case(3)
    g = rend.render_backward(scene, lab, front_camera(32, 32, 60.0), RasterConfig())
    assert all(np.all(v == 0) for v in g.values())


@pytest.mark.parametrize("case", ["topk4", "full"])
def test_gpu_backward_vs_compiled_reference(rend, case):
    """The GPU backward against THE REFERENCE'S OWN pipeline_backward (pipeline.cpp, compiled unchanged in
    oracle/_ref) on a query-free scene without a SOGMM model and l_iso = 0: the upstream colour plane is
    the reference's loss_rgb_backward, the semantic plane its clamped cross-entropy (restated in
    tests/test_ref_pin.py); every surfel gradient within fp64 summation-order noise."""
    from oracle import pyref as R
    from tests.test_ref_pin import _pose_cameras, sem_ce_plane_grad
    if not R.available():
        pytest.skip("oracle/_ref not built")
    sc, _, cam = make_street_scene(StreetSpec(n_surfels=3000, image_w=96, image_h=64, c_sem=6), with_labels=False)
    rs = R.RefScene(sc.surfels, sc.f_sem, None)
    rng = np.random.default_rng(3)
    rgb = rng.uniform(0, 1, (64, 96, 3))
    sem = rng.integers(-1, 6, (64, 96)).astype(np.int32)
    cfg = RasterConfig(blending=Blending.TopK, top_k=4) if case == "topk4" else RasterConfig()
    try:
        for c in (cam, _pose_cameras(96, 64)[4]):
            r = rs.pipeline_backward(c, cfg, rgb, sem, l_sem=0.5, l_iso=0.0)
            g_sem = sem_ce_plane_grad(rs.render(c, cfg)["sem_feat"], sem, 0.5)
            g = rend.render_backward(sc, None, c, cfg, r["g_color_plane"], g_sem, None)
            for k in ("opacity", "color", "f_sem", "center", "rotation", "scales"):
                scale = max(np.max(np.abs(r[k])), 1e-300)
                assert np.max(np.abs(g[k] - r[k])) <= 1e-9 * scale, k
    finally:
        rs.close()


@pytest.mark.parametrize("blending,k", [(Blending.Full, 16), (Blending.TopK, 2)])
def test_gpu_backward_ragged_image(rend, blending, k):
    """An image whose sides are not multiples of the 8x4 list blocks (block-major cache lists with
    partial blocks at the right and bottom edges)."""
    scene, lab = scene_case(7)
    cam = front_camera(37, 29, 50.0)
    cfg = RasterConfig(blending=blending, top_k=k)
    rng = np.random.default_rng(4)
    gc, gs, gi = rng.normal(size=(29, 37, 3)), rng.normal(size=(29, 37, 3)), rng.normal(size=(29, 37, 2))
    assert_grads_close(rend.render_backward(scene, lab, cam, cfg, gc, gs, gi),
                       O.render_backward(scene, lab, cam, cfg, gc, gs, gi))
