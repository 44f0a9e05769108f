"""GPU parity of the panoptic rows through the C-ABI against the
oracle: assign_labels (panoptic.cpp:36-91) bit-exact in dist and argmax; render_panoptic
(metrics.cpp:339-369) bit-exact in ids, classes and semantic classes (the blend sums
features and labels in fp64 in blend order, as raster.cpp:456-499)."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2604_10982_b200 import (Binning, Blending, InstanceQuery, RasterConfig, Renderer, SceneMap, StreetSpec,
                                   density_scale, make_street_scene, street_f_ins, street_queries)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rend():
    r = Renderer(0)
    yield r
    r.close()


@pytest.fixture(scope="module")
def street():
    spec = StreetSpec(n_surfels=12000, image_w=256, image_h=192, c_sem=32, seed=7)
    scene, _, cam = make_street_scene(spec, with_labels=False)
    f_ins = street_f_ins(spec)
    qs = street_queries(24, c_ins=8)
    qs[5].alive = False
    qs[17].alive = False
    return SceneMap(scene.surfels, scene.f_sem, f_ins, qs), cam


def test_street_f_ins_shape(street):
    sc, _ = street
    assert sc.f_ins.shape == (len(sc), 8)
    assert abs(np.std(sc.f_ins) - 0.3) < 0.01  # 0.3 N(0,1) (synthetic.cpp:283-284)


def test_gpu_assign_labels_bit_exact(rend, street):
    sc, _ = street
    ds = rend.upload(sc, None, exact=True)
    gd, ga = rend.assign_labels(ds, sc.queries)
    od, oa = O.assign_labels(sc.surfels, sc.f_ins, sc.queries)
    assert np.array_equal(ga, oa)
    assert np.array_equal(gd.view(np.uint64), od.view(np.uint64))
    assert np.all(gd[:, 5] == 0) and np.all(gd[:, 17] == 0)


def test_gpu_assign_labels_kat(rend):
    # test_panoptic.cpp:93-112 through the GPU
    s = np.zeros((6, 13))
    s[:, 0] = np.arange(6) * 0.3
    s[:, 3] = 1.0
    s[:, 7:9] = 0.1
    f = np.array([[0.1 * i, -0.2] for i in range(6)])
    sc = SceneMap(s, None, f)
    ds = rend.upload(sc, None, exact=True)
    q = InstanceQuery(np.array([1.0, 1.0]), np.zeros(3), np.eye(3))
    d, a = rend.assign_labels(ds, [q])
    assert np.allclose(d[:, 0], 1.0, atol=1e-12) and np.all(a == 0)
    d, a = rend.assign_labels(ds, [q, InstanceQuery(np.array([1.0, 1.0]), np.zeros(3), np.eye(3))])
    assert np.allclose(d, 0.5, atol=1e-12) and np.all(a == 0)
    dead = InstanceQuery(np.array([1.0, 1.0]), np.zeros(3), np.eye(3), alive=False)
    d, a = rend.assign_labels(ds, [dead])
    assert np.all(d == 0) and np.all(a == -1)


@pytest.mark.parametrize("blending,k", [(Blending.TopK, 16), (Blending.TopK, 8), (Blending.Full, 16)])
def test_gpu_render_panoptic_bit_exact(rend, street, blending, k):
    sc, cam = street
    cfg = RasterConfig(binning=Binning.Ellipse, blending=blending, top_k=k)
    g = rend.render_panoptic_scene(sc, cam, cfg)
    o = O.render_panoptic(sc, sc.f_ins, sc.queries, cam, cfg)
    assert np.array_equal(g.ids, o["ids"]), "ids"
    assert np.array_equal(g.classes, o["classes"]), "classes"
    assert np.array_equal(g.sem_classes, o["sem_classes"]), "sem_classes"
    assert (g.ids >= 0).mean() > 0.3  # a populated frame


def test_gpu_render_panoptic_no_queries_and_no_features(rend, street):
    sc, cam = street
    bare = SceneMap(sc.surfels, None)
    ds = rend.upload(bare, None, exact=True)
    pr = rend.render_panoptic(ds, cam, RasterConfig(), [])
    o = O.render_panoptic(bare, np.zeros((len(bare), 0)), [], cam, RasterConfig())
    assert np.all(pr.ids == -1) and np.all(pr.classes == -1) and np.all(pr.sem_classes == -1)
    assert np.array_equal(pr.ids, o["ids"]) and np.array_equal(pr.sem_classes, o["sem_classes"])


def test_gpu_render_panoptic_needs_exact_scene(rend, street):
    sc, cam = street
    ds = rend.upload(sc)  # features, no labels, no PSM_SCENE_EXACT_FEATURES: fp32 rows only
    with pytest.raises(NotImplementedError):  # PSM_EUNSUPPORTED
        rend.render_panoptic(ds, cam, RasterConfig(), [0, 1])
    # a scene with labels keeps its fp64 rows (the render's exact label phase), so it also serves render_panoptic
    lab = np.tile(np.array([0.25, 0.75]), (len(sc), 1))
    a = rend.render_panoptic(rend.upload(sc, lab), cam, RasterConfig(), [3, 4])
    b = rend.render_panoptic(rend.upload(sc, lab, exact=True), cam, RasterConfig(), [3, 4])
    for k in ("ids", "classes", "sem_classes"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


def test_gpu_render_panoptic_c3p_full_size(rend):
    # C3p: 1M surfels, 1280x720, 64-d semantics, N_q = 32 queries, K = 8
    spec = StreetSpec(n_surfels=1_000_000, image_w=1280, image_h=720, c_sem=64, seed=7,
                      scale_mult=density_scale(1_000_000, 1280, 720))
    scene, _, cam = make_street_scene(spec, with_labels=False)
    sc = SceneMap(scene.surfels, scene.f_sem, street_f_ins(spec), street_queries(32))
    cfg = RasterConfig(binning=Binning.Ellipse, blending=Blending.TopK, top_k=8)
    g = rend.render_panoptic_scene(sc, cam, cfg)
    o = O.render_panoptic(sc, sc.f_ins, sc.queries, cam, RasterConfig(binning=Binning.Aabb, blending=Blending.TopK,
                                                                       top_k=8))
    assert np.array_equal(g.ids, o["ids"])
    assert np.array_equal(g.classes, o["classes"])
    assert np.array_equal(g.sem_classes, o["sem_classes"])
    # and directly against THE REFERENCE'S OWN render_panoptic (metrics.cpp:339-369 with
    # panoptic.cpp's assign_labels and raster.cpp's render, compiled unchanged in oracle/_ref)
    from oracle import pyref as R
    if R.available():
        r = R.render_panoptic(sc, cam, RasterConfig(binning=Binning.Aabb, blending=Blending.TopK, top_k=8))
        for k in ("ids", "classes", "sem_classes"):
            assert np.array_equal(getattr(g, k), r[k]), k


@pytest.mark.parametrize("c_sem,n_q", [(8, 16), (64, 40), (128, 64), (256, 100), (3, 5), (7, 4), (33, 30), (61, 40)])
@pytest.mark.parametrize("blending,k", [(Blending.TopK, 8), (Blending.TopK, 32), (Blending.Full, 16)])
def test_gpu_render_panoptic_feature_widths(rend, c_sem, n_q, blending, k):
    """The fp64 panoptic phase at every lane shape (8 lanes per pixel up to 96 channels, 16 up to 128,
    32 beyond; odd widths; Top-K rounds beyond the lanes of a pixel), ids / classes / semantic classes
    bit-exact vs the oracle."""
    spec = StreetSpec(n_surfels=4000, image_w=128, image_h=96, c_sem=c_sem, seed=11)
    scene, _, cam = make_street_scene(spec, with_labels=False)
    qs = street_queries(n_q, c_ins=8)
    sc = SceneMap(scene.surfels, scene.f_sem, street_f_ins(spec), qs)
    cfg = RasterConfig(binning=Binning.Ellipse, blending=blending, top_k=k)
    g = rend.render_panoptic_scene(sc, cam, cfg)
    o = O.render_panoptic(sc, sc.f_ins, sc.queries, cam, cfg)
    for key in ("ids", "classes", "sem_classes"):
        assert np.array_equal(getattr(g, key), o[key]), key
