"""GPU parity: the sm_100a path (through the C-ABI, libpsm.so) against the CPU oracle on the same
seeded inputs. Bit-exact: sorted (tile, depth-rank) keys, tile lists, per-tile ranges, depth order,
Top-K source sets, blend counts, RN-Total / blended_total / n_proj. Within 1e-4 absolute (the
north-star tolerance): colour, depth, normal, alpha, semantic-feature and label planes."""
import ctypes as C
import math

import numpy as np
import pytest

from oracle import pyoracle as O
from oracle import pyref as R
from paper_2604_10982_b200 import (Binning, Blending, RasterConfig, Renderer, RenderTargets, SceneMap, StreetSpec,
                                   density_scale, make_street_scene, trajectory_cameras)
from paper_2604_10982_b200 import _abi as A
from tests.helpers import Rng, facing_surfel, front_camera, scene_of

pytestmark = pytest.mark.gpu
ATOL = 1e-4  # north-star tolerance for fp32 planes


@pytest.fixture(scope="module")
def rend():
    r = Renderer(0)
    yield r
    r.close()


def gpu_render(rend, scene, labels, cam, cfg, debug=True):
    out = RenderTargets()
    dbg = None
    arrs = {}
    if debug:
        ref = O.render(scene, labels, cam, cfg, planes=False)  # sizes for the debug buffers
        rn, n_proj = ref["counters"]["rn_total"], ref["counters"]["n_proj"]
        tiles = ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
        k = max(cfg.top_k, 1)
        arrs = {"tile_keys": np.zeros(max(rn, 1), np.uint64), "tile_vals": np.zeros(max(rn, 1), np.int32),
                "tile_ranges": np.zeros((tiles, 2), np.int32), "depth_order": np.zeros(max(n_proj, 1), np.int32),
                "topk_src": np.full((cam.height, cam.width, k), -1, np.int32)}
        p = lambda a: a.ctypes.data_as(C.c_void_p)
        dbg = A.psm_debug(p(arrs["tile_keys"]), p(arrs["tile_vals"]), rn, p(arrs["tile_ranges"]),
                          p(arrs["depth_order"]), n_proj, p(arrs["topk_src"]))
    rend.render_into(out, scene, labels, cam, cfg, debug=dbg)
    if debug:
        arrs["tile_keys"] = arrs["tile_keys"][:out.rn_total]
        arrs["tile_vals"] = arrs["tile_vals"][:out.rn_total]
        arrs["depth_order"] = arrs["depth_order"][:out.n_proj]
    return out, arrs


def assert_parity(rend, scene, labels, cam, cfg, check_debug=True):
    g, gd = gpu_render(rend, scene, labels, cam, cfg, debug=check_debug)
    o = O.render(scene, labels, cam, cfg, debug=check_debug)
    oc = o["counters"]
    # counters (raster.hpp:36-37,65)
    assert g.rn_total == oc["rn_total"]
    assert g.n_proj == oc["n_proj"]
    assert g.blended_total == oc["blended_total"]
    assert g.rn_per_tile == pytest.approx(oc["rn_per_tile"], rel=0, abs=0)
    if check_debug:
        assert np.array_equal(gd["depth_order"], o["depth_order"]), "depth order"
        assert np.array_equal(gd["tile_ranges"], o["tile_ranges"]), "tile ranges"
        assert np.array_equal(gd["tile_vals"], o["tile_vals"]), "tile lists"
        assert np.array_equal(gd["tile_keys"], o["tile_keys"]), "sorted keys"
        if cfg.blending == Blending.TopK:
            gs = np.sort(np.where(gd["topk_src"] < 0, np.iinfo(np.int32).max, gd["topk_src"]), axis=-1)
            os_ = np.sort(np.where(o["topk_src"] < 0, np.iinfo(np.int32).max, o["topk_src"]), axis=-1)
            assert np.array_equal(gs, os_), "Top-K source sets"
    assert np.array_equal(g.blend_count, o["blend_count"]), "blend_count"
    for k in ("color", "depth", "normal", "alpha_acc", "sem_feat", "ins_dist"):
        a, b = getattr(g, k), o[k]
        assert a.shape == b.shape, k
        if a.size:
            err = np.max(np.abs(a.astype(np.float64) - b))
            assert err <= ATOL, (k, err)
    # ins_argmax: exact (labels blend in fp64 in blend order, raster.cpp:456-498)
    assert np.array_equal(g.ins_argmax, o["ins_argmax"]), "ins_argmax"
    return g, o


# ------------------------------------------------------------ test_raster.cpp KATs through the GPU
def test_gpu_single_opaque_surfel(rend):
    cam = front_camera()
    sc = scene_of([facing_surfel((0, 0, 2), 0.2, 0.2, 1.0, (0.3, 0.6, 0.9))])
    g, _ = assert_parity(rend, sc, None, cam, RasterConfig(background=(0.1, 0.1, 0.1)))
    x, y = int(cam.cx), int(cam.cy)
    assert np.allclose(g.color[y, x], (0.3, 0.6, 0.9), atol=1e-6)
    assert abs(g.alpha_acc[y, x, 0] - 1.0) < 1e-6
    assert abs(g.depth[y, x, 0] - 2.0) < 1e-5 and abs(g.depth[y, x, 1] - 2.0) < 1e-5


def test_gpu_single_entry_tiles_after_dense_frame(rend):
    """Tiles holding exactly one (surfel, tile) entry (no sort needed) must still get that entry's
    source id and warp-block mask, also when the context's buffers hold a previous frame's lists."""
    sc, _, cam = make_street_scene(StreetSpec(n_surfels=3000, image_w=128, image_h=96, c_sem=0), with_labels=False)
    assert_parity(rend, sc, None, cam, RasterConfig())  # fills the key/list buffers with other data
    cam = front_camera(128, 96)
    # small surfels far apart (each alone in its tiles), placed so that their ids are non-zero
    far = [facing_surfel((0, 0, -5), 0.2, 0.2, 1.0, (1, 1, 1))] * 3  # culled (behind the camera)
    iso = [facing_surfel((dx, dy, 4), 0.05, 0.05, 0.9, (0.2 + 0.1 * i, 0.5, 0.7))
           for i, (dx, dy) in enumerate([(-1.5, -1.0), (0.0, 0.0), (1.6, 1.1), (1.5, -1.2)])]
    for binning in (Binning.Circle, Binning.Aabb, Binning.Ellipse):
        g, _ = assert_parity(rend, scene_of(far + iso), None, cam, RasterConfig(binning=binning))
        assert np.count_nonzero(g.blend_count) > 0


def test_gpu_two_surfel_alpha_arithmetic(rend):
    cam = front_camera()
    sc = scene_of([facing_surfel((0, 0, 2), 0.2, 0.2, 0.5, (1, 0, 0)),
                   facing_surfel((0, 0, 3), 0.3, 0.3, 1.0, (0, 1, 0))])
    g, _ = assert_parity(rend, sc, None, cam, RasterConfig())
    x, y = int(cam.cx), int(cam.cy)
    assert np.allclose(g.color[y, x], (0.5, 0.5, 0.0), atol=1e-6)


def test_gpu_empty_scene(rend):
    cam = front_camera(16, 16)
    g = rend.render(SceneMap(np.zeros((0, 13))), None, cam, RasterConfig(background=(0.25, 0.5, 0.75)))
    assert np.all(g.color == np.array([0.25, 0.5, 0.75], np.float32))
    assert np.all(g.alpha_acc == 0) and np.all(g.ins_argmax == -1) and np.all(g.blend_count == 0)
    assert g.blended_total == 0 and g.rn_total == 0


def test_gpu_degenerate_quaternion_raises(rend):
    cam = front_camera()
    bad = facing_surfel((0, 0, 2), 0.2, 0.2, 1.0, (1, 1, 1), quat=(0, 0, 0, 0))
    with pytest.raises(ValueError):
        rend.render(scene_of([bad]), None, cam, RasterConfig())
    # behind the camera the reference never reaches rotation_from_quat (raster.cpp:97-99)
    behind = facing_surfel((0, 0, -2), 0.2, 0.2, 1.0, (1, 1, 1), quat=(0, 0, 0, 0))
    rend.render(scene_of([behind]), None, cam, RasterConfig())


# ------------------------------------------------------------ street scenes
@pytest.fixture(scope="module")
def c0():  # acceptance standard street (acceptance.cpp:33-42): 12k surfels, 256x192, C_sem 32, 256 labels
    return make_street_scene(StreetSpec(n_surfels=12000, image_w=256, image_h=192, c_sem=32, seed=7))


@pytest.mark.parametrize("binning", [Binning.Circle, Binning.Aabb, Binning.Ellipse])
@pytest.mark.parametrize("blending", [Blending.Full, Blending.TopK])
def test_gpu_c0_grid(rend, c0, binning, blending):
    sc, labels, cam = c0
    assert_parity(rend, sc, labels, cam, RasterConfig(binning=binning, blending=blending, top_k=16))


def test_gpu_c1_rgb_depth(rend):
    sc, _, cam = make_street_scene(StreetSpec(n_surfels=10000, image_w=256, image_h=256, c_sem=0))
    assert_parity(rend, sc, None, cam, RasterConfig(binning=Binning.Aabb))


@pytest.mark.parametrize("k", [1, 5, 8, 16, 32])
def test_gpu_topk_sizes(rend, k):
    sc, _, cam = make_street_scene(StreetSpec(n_surfels=3000, image_w=128, image_h=96, c_sem=64,
                                              scale_mult=density_scale(3000, 128, 96)))
    assert_parity(rend, sc, None, cam, RasterConfig(binning=Binning.Ellipse, blending=Blending.TopK, top_k=k))


@pytest.mark.parametrize("variant", ["no_cutoff", "no_depth_normal", "background", "t_min0", "ragged", "chi2"])
def test_gpu_config_variants(rend, variant):
    w, h = (100, 70) if variant == "ragged" else (96, 64)
    sc, labels, cam = make_street_scene(StreetSpec(n_surfels=1500, image_w=w, image_h=h, c_sem=8, n_instances=12))
    cfg = {
        "no_cutoff": RasterConfig(support_cutoff=False, binning=Binning.Ellipse),  # Ellipse falls back to AABB
        "no_depth_normal": RasterConfig(render_depth_normal=False, blending=Blending.TopK, top_k=4),
        "background": RasterConfig(background=(0.2, 0.4, 0.6), binning=Binning.Circle),
        "t_min0": RasterConfig(t_min=0.0, blending=Blending.TopK, top_k=8),
        "ragged": RasterConfig(binning=Binning.Ellipse, blending=Blending.TopK, top_k=8),
        "chi2": RasterConfig(chi2=4.0, binning=Binning.Ellipse),
    }[variant]
    assert_parity(rend, sc, labels, cam, cfg)


def test_gpu_random_surfels(rend):
    rng = Rng(17)
    rows = []
    for _ in range(600):
        c = (rng.uniform(-1.2, 1.2), rng.uniform(-1, 1), rng.uniform(0.5, 6))
        q = rng.unit_quaternion()
        rows.append(facing_surfel(c, rng.uniform(0.01, 0.6), rng.uniform(0.01, 0.6), rng.uniform(0.05, 1.0),
                                  (rng.uniform(), rng.uniform(), rng.uniform()), quat=q))
    f = np.array([[rng.normal() for _ in range(40)] for _ in rows])
    sc = SceneMap(np.array(rows), f)
    cam = front_camera(160, 120, 120.0)
    for cfg in (RasterConfig(binning=Binning.Ellipse, blending=Blending.TopK, top_k=8),
                RasterConfig(binning=Binning.Circle, blending=Blending.Full)):
        assert_parity(rend, sc, None, cam, cfg)


def test_gpu_extreme_footprints(rend):
    """Needles, grazing views, sub-pixel and near-plane (huge) surfels, centres far off-screen
    with footprints reaching in, on a ragged image: stresses the fp32 warp-block masks (their
    margins must never drop a candidate whose fp64 support test passes) and the tile rows."""
    rng = Rng(23)
    rows = []
    for i in range(900):
        kind = i % 6
        if kind == 0:    # needles at random orientation
            c = (rng.uniform(-1, 1), rng.uniform(-0.8, 0.8), rng.uniform(1, 5))
            s1, s2 = rng.uniform(0.3, 2.0), rng.uniform(0.0005, 0.003)
        elif kind == 1:  # nearly edge-on to the camera
            c = (rng.uniform(-1, 1), rng.uniform(-0.8, 0.8), rng.uniform(1, 5))
            s1, s2 = rng.uniform(0.05, 0.5), rng.uniform(0.05, 0.5)
        elif kind == 2:  # sub-pixel
            c = (rng.uniform(-1, 1), rng.uniform(-0.8, 0.8), rng.uniform(2, 8))
            s1, s2 = rng.uniform(0.0005, 0.004), rng.uniform(0.0005, 0.004)
        elif kind == 3:  # close to the near plane: footprints far larger than the image
            c = (rng.uniform(-0.3, 0.3), rng.uniform(-0.3, 0.3), rng.uniform(0.12, 0.4))
            s1, s2 = rng.uniform(0.05, 0.3), rng.uniform(0.01, 0.3)
        elif kind == 4:  # centre well off-screen, large enough to reach in
            c = (rng.uniform(2.0, 4.0) * (1 if rng.uniform() < 0.5 else -1), rng.uniform(-1, 1), rng.uniform(1.5, 3))
            s1, s2 = rng.uniform(1.0, 3.0), rng.uniform(0.05, 1.0)
        else:            # ordinary
            c = (rng.uniform(-1, 1), rng.uniform(-0.8, 0.8), rng.uniform(1, 6))
            s1, s2 = rng.uniform(0.02, 0.3), rng.uniform(0.02, 0.3)
        q = rng.unit_quaternion()
        if kind == 1:  # rotate about y by ~90 degrees: the surfel plane almost contains the view ray
            a = math.pi / 2 * rng.uniform(0.97, 0.999) / 2
            q = (math.cos(a), 0.0, math.sin(a), 0.0)
        rows.append(facing_surfel(c, s1, s2, rng.uniform(0.2, 1.0), (rng.uniform(), rng.uniform(), rng.uniform()),
                                  quat=q))
    sc = SceneMap(np.array(rows), np.array([[rng.normal() for _ in range(32)] for _ in rows]))
    cam = front_camera(100, 70, 90.0)
    for cfg in (RasterConfig(binning=Binning.Ellipse, blending=Blending.TopK, top_k=8),
                RasterConfig(binning=Binning.Aabb, blending=Blending.Full),
                RasterConfig(binning=Binning.Circle, blending=Blending.TopK, top_k=16, chi2=16.0)):
        g, _ = assert_parity(rend, sc, None, cam, cfg)
        assert g.blended_total > 0


def test_gpu_permutation_bit_identical(rend):
    sc, labels, cam = make_street_scene(StreetSpec(n_surfels=2000, image_w=96, image_h=64, c_sem=3,
                                                   n_instances=8))
    perm = np.random.default_rng(3).permutation(len(sc))
    sh = SceneMap(sc.surfels[perm], sc.f_sem[perm])
    cfg = RasterConfig(blending=Blending.TopK, top_k=8)
    a = rend.render(sc, labels, cam, cfg)
    b = rend.render(sh, labels[perm], cam, cfg)
    for k in ("color", "depth", "normal", "blend_count", "alpha_acc"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


# ------------------------------------------------------------ full-size C3 (the bench workload)
@pytest.fixture(scope="module")
def c3():
    n, w, h = 1_000_000, 1280, 720
    return make_street_scene(StreetSpec(n_surfels=n, image_w=w, image_h=h, c_sem=64,
                                        scale_mult=density_scale(n, w, h)), with_labels=False)


def test_gpu_c3_full_size_parity(rend, c3):
    """1M surfels, 1280x720, 64-d features, Top-K = 8, Ellipse binning: every bit-exact artefact and
    every plane against the oracle at the benchmark's own size."""
    sc, _, cam = c3
    g, o = assert_parity(rend, sc, None, cam, RasterConfig(binning=Binning.Ellipse, blending=Blending.TopK,
                                                          top_k=8))
    assert g.rn_total > 1_000_000


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
def test_gpu_c3_full_size_vs_compiled_reference(rend, c3):
    """The GPU frame against THE REFERENCE'S OWN render_into (oracle/_ref: raster.cpp compiled unchanged)
    at the metric's config, the street camera and a C5 trajectory pose: blend counts, ins_argmax and
    blended_total exact, every fp32 plane within the north star's 1e-4 of the reference's fp64 plane.
    The reference bins by AABB, the GPU by ellipse (identical planes, test above)."""
    sc, _, cam = c3
    rs = R.RefScene(sc.surfels, sc.f_sem, None)
    try:
        for c in (cam, trajectory_cameras(256, 1280, 720, first=200, count=1)[0]):
            g = rend.render(sc, None, c, RasterConfig(binning=Binning.Ellipse, blending=Blending.TopK, top_k=8))
            r = rs.render(c, RasterConfig(binning=Binning.Aabb, blending=Blending.TopK, top_k=8, threads=0))
            assert g.blended_total == r["blended_total"]
            assert np.array_equal(g.blend_count, r["blend_count"]) and np.array_equal(g.ins_argmax, r["ins_argmax"])
            for k in ("color", "depth", "normal", "alpha_acc", "sem_feat"):
                err = np.max(np.abs(getattr(g, k).astype(np.float64) - r[k]))
                assert err <= ATOL, (k, err)
    finally:
        rs.close()


def test_gpu_c3_binning_output_identity(rend, c3):
    """Size-independent property at full size: Circle, AABB and Ellipse binning give bit-identical
    planes (support cutoff on), RN-Total strictly decreasing."""
    sc, _, cam = c3
    outs = [rend.render(sc, None, cam, RasterConfig(binning=b, blending=Blending.TopK, top_k=8))
            for b in (Binning.Circle, Binning.Aabb, Binning.Ellipse)]
    for o in outs[1:]:
        for k in ("color", "depth", "normal", "sem_feat", "blend_count", "alpha_acc"):
            assert np.array_equal(getattr(outs[0], k), getattr(o, k)), k
        assert o.blended_total == outs[0].blended_total
    assert outs[0].rn_total > outs[1].rn_total > outs[2].rn_total
    bc = outs[0].blend_count
    assert outs[0].blended_total == int(np.minimum(bc, 8).sum())
    assert np.all(outs[0].alpha_acc >= 0) and np.all(outs[0].alpha_acc <= 1)


@pytest.mark.parametrize("count", [5000, 20000])
def test_gpu_huge_buckets_and_depth_ties(rend, count):
    """Buckets beyond the 4096 and 16384 shared-memory sort classes (the merge-path global passes), with
    exact depth ties broken by source index (raster.cpp:78-83)."""
    rng = np.random.default_rng(count)
    cam = front_camera(48, 48, 60.0)
    z = rng.choice(np.linspace(2.0, 6.0, count // 4), size=count)  # every depth shared by ~4 surfels
    z[::3] = np.nextafter(z[::3], np.inf)  # 1-ulp neighbours: equal truncated sort keys, different depths
    xy = rng.uniform(-0.02, 0.02, size=(count, 2)) * z[:, None]
    rows = np.zeros((count, 13))
    rows[:, 0:2] = xy
    rows[:, 2] = z
    rows[:, 3] = 1.0
    rows[:, 7] = rng.uniform(0.005, 0.02, count) * z
    rows[:, 8] = rng.uniform(0.005, 0.02, count) * z
    rows[:, 9] = rng.uniform(0.02, 0.1, count)
    rows[:, 10:13] = rng.uniform(0, 1, (count, 3))
    sc = SceneMap(rows, rng.standard_normal((count, 8)))
    g, o = assert_parity(rend, sc, None, cam, RasterConfig(binning=Binning.Aabb, blending=Blending.TopK, top_k=8))
    tiles = O.bin_surfels(rows, cam, RasterConfig(), 1)["tiles"]
    assert max(len(t) for t in tiles) > (16384 if count > 16384 else 4096)


def test_gpu_ins_argmax_below_fp32_resolution(rend):
    """Label masses that differ only below fp32 resolution: the argmax follows the fp64 blend-order sums
    (raster.cpp:486-498), including exact fp64 ties (first index wins)."""
    sc, _, cam = make_street_scene(StreetSpec(n_surfels=2500, image_w=96, image_h=64, c_sem=5, n_instances=4))
    n = len(sc)
    rng = np.random.default_rng(11)
    base = rng.uniform(0.1, 0.4, n)
    labels = np.stack([base, base + 1e-12 * (1 + (np.arange(n) % 3)), base, rng.uniform(0, 0.05, n)], axis=1)
    labels[::7, 1] = labels[::7, 0]  # exact ties on some surfels
    for cfg in (RasterConfig(blending=Blending.TopK, top_k=8, binning=Binning.Ellipse),
                RasterConfig(blending=Blending.Full)):
        g, o = assert_parity(rend, sc, labels, cam, cfg)
        assert np.count_nonzero(o["ins_argmax"] == 1) > 0
