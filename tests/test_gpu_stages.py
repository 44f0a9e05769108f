"""GPU parity of the stage entry points (include/psm.h; reference raster.hpp:87-126) and of
RenderCache (raster.hpp:76-82) against the oracle, which tests/test_ref_pin.py pins bit for bit
to the reference's own compiled code:
  project_surfel (raster.cpp:94-142), bin_circle / bin_aabb (:51-90,144-152),
  sample_surfel_alpha / evaluate_alpha (:154-177), topk_select (:225-251), and render with a
  RenderCache (:310-315,399-403): projected list, tile grid, per-pixel contributors."""
import math

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2604_10982_b200 import (Binning, Blending, Camera, RasterConfig, Renderer, SceneMap, StreetSpec,
                                   make_street_scene, trajectory_cameras)
from paper_2604_10982_b200 import stages as S
from tests.helpers import Rng, facing_surfel, front_camera
from tests.test_gpu_poses_shapes import make_pose

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rend():
    r = Renderer(0)
    yield r
    r.close()


def random_surfels(n, seed):
    rng = Rng(seed)
    rows = []
    for _ in range(n):
        q = rng.unit_quaternion()
        rows.append([rng.uniform(-3, 3), rng.uniform(-2, 2), rng.uniform(-1, 25), *q, rng.uniform(0.01, 1.5),
                     rng.uniform(0.01, 0.4), rng.uniform(0.1, 1), rng.uniform(), rng.uniform(), rng.uniform()])
    return np.array(rows)


def cams():
    return [front_camera(160, 120, 120.0), trajectory_cameras(256, 320, 240, first=70, count=1)[0],
            make_pose(320, 240)]


def test_gpu_project_surfel_bit_exact(rend):
    s = random_surfels(3000, 5)
    cfg = RasterConfig()
    for cam in cams():
        arr, status = S.project_surfels(s, cam, cfg, renderer=rend)
        for i in range(len(s)):
            o = O.project_surfel(s[i], cam, cfg.chi2)
            assert bool(status[i]) == (o is not None), i
            if o is None:
                continue
            g = S.ProjectedSurfel.from_c(arr[i])
            assert g.source == -1
            for k in ("sigma", "h", "h_inv", "footprint_inv", "normal_vis"):
                assert np.array_equal(getattr(g, k), o[k]), (i, k)
            assert np.array_equal(g.screen_center, o["center"]) and g.sort_depth == o["sort_depth"]


def test_gpu_project_surfel_degenerate_quaternion(rend):
    bad = facing_surfel((0, 0, 2), 0.2, 0.2, 1.0, (1, 1, 1), quat=(0, 0, 0, 0))
    with pytest.raises(ValueError):
        S.project_surfel(bad, front_camera(), RasterConfig(), renderer=rend)
    behind = facing_surfel((0, 0, -2), 0.2, 0.2, 1.0, (1, 1, 1), quat=(0, 0, 0, 0))
    assert S.project_surfel(behind, front_camera(), RasterConfig(), renderer=rend) is None  # raster.cpp:97-99


@pytest.mark.parametrize("binning", [Binning.Circle, Binning.Aabb])
def test_gpu_bin_bit_exact(rend, binning):
    """Tile lists (projected indices in (depth, source) order) and RN counters, also with a chi2 for the
    AABB box that differs from the config's (bin_aabb's own argument) and a 32-px tile."""
    sc, _, cam0 = make_street_scene(StreetSpec(n_surfels=12000, image_w=256, image_h=192, c_sem=0))
    for cam in (cam0, trajectory_cameras(256, 256, 192, first=31, count=1)[0]):
        for cfg, chi2 in ((RasterConfig(binning=binning), 9.0), (RasterConfig(binning=binning, tile_size=32), 4.0)):
            arr, status = S.project_surfels(sc.surfels, cam, cfg, renderer=rend)
            idx = np.flatnonzero(status)
            proj = (type(arr[0]) * len(idx))()
            for j, i in enumerate(idx):
                proj[j] = arr[i]
                proj[j].source = int(i)
            g = (S.bin_circle(proj, cam, cfg, renderer=rend) if binning == Binning.Circle
                 else S.bin_aabb(proj, cam, cfg, chi2, renderer=rend))
            o = O.bin_surfels(sc.surfels, cam, cfg, int(binning), chi2=chi2 if binning == Binning.Aabb else None)
            assert g.rn_total == o["rn_total"] and g.rn_per_tile == o["rn_per_tile"]
            for t, (a, b) in enumerate(zip(g.tiles, o["tiles"])):
                assert np.array_equal(idx[a], b), t  # projected index -> source == the oracle's source ids


def test_gpu_bin_source_order_ties(rend):
    """Equal sort depths are ordered by source, also when the projected list is not in source order."""
    rows = [facing_surfel((0.01 * i, 0, 3.0), 0.3, 0.3, 0.5, (1, 1, 1)) for i in range(40)]
    cam = front_camera(64, 64)
    arr, status = S.project_surfels(np.array(rows), cam, RasterConfig(), renderer=rend)
    perm = np.random.default_rng(2).permutation(40)
    proj = (type(arr[0]) * 40)()
    for j, i in enumerate(perm):
        proj[j] = arr[i]
        proj[j].source = int(i)
    g = S.bin_aabb(proj, cam, RasterConfig(), 9.0, renderer=rend)
    for lst in g.tiles:
        assert list(perm[lst]) == sorted(perm[lst])


def test_gpu_sample_and_evaluate_alpha(rend):
    s = random_surfels(400, 9)
    rng = Rng(3)
    for cfg in (RasterConfig(), RasterConfig(support_cutoff=False, alpha_min=0.05)):
        for cam in cams():
            arr, status = S.project_surfels(s, cam, cfg, renderer=rend)
            idx = np.flatnonzero(status)
            qi, px, py, src = [], [], [], []
            for i in idx:
                c = arr[i].screen_center
                for _ in range(3):
                    qi.append(i)
                    px.append(math.floor(c[0] + rng.uniform(-6, 6)) + 0.5)
                    py.append(math.floor(c[1] + rng.uniform(-6, 6)) + 0.5)
            g = S.sample_alpha(arr, s[:, 9], qi, px, py, cam, cfg, renderer=rend)
            for q in range(len(qi)):
                o = O.evaluate_alpha(s[qi[q]], cam, px[q], py[q], cfg)
                assert g[q]["alpha"] == o["alpha"] and bool(g[q]["inside"]) == o["inside"], q
                if o["inside"]:
                    assert g[q]["u"] == o["u"] and g[q]["v"] == o["v"] and g[q]["w2"] == o["w2"]


def test_gpu_topk_select(rend):
    rng = np.random.default_rng(7)
    lists, offs = [], [0]
    for m in (0, 1, 3, 8, 9, 17, 40, 100):
        w = rng.uniform(0, 1, m)
        w[: m // 4] = w[0] if m else w[: m // 4]  # exact ties, broken by proj ascending
        p = rng.integers(0, 50, m).astype(np.int32)
        lists.append((w, p))
        offs.append(offs[-1] + m)
    W = np.concatenate([l[0] for l in lists]) if lists else np.zeros(0)
    P = np.concatenate([l[1] for l in lists]).astype(np.int32)
    for k in (1, 4, 8, 16, 64):
        g = S.topk_select_lists(W, P, offs, k, renderer=rend)
        for li, (w, p) in enumerate(lists):
            o = O.topk_select(w, p, k)
            assert np.array_equal(g[offs[li]:offs[li + 1]], o), (k, li)


@pytest.mark.parametrize("blending", [Blending.Full, Blending.TopK])
def test_gpu_render_cache(rend, blending):
    """RenderCache::pixels (raster.cpp:399-403) bit for bit: per pixel, the contributors in blend order
    with their alpha; projected surfels in source order; planes as psm_render's."""
    sc, labels, cam = make_street_scene(StreetSpec(n_surfels=4000, image_w=128, image_h=96, c_sem=6,
                                                   n_instances=5))
    for c in (cam, make_pose(128, 96)):
        cfg = RasterConfig(blending=blending, top_k=8)
        cache = S.RenderCache()
        g = S.render_cached(sc, labels, c, cfg, cache, renderer=rend)
        o = O.render_cache(sc, labels, c, cfg)
        plain = rend.render(sc, labels, c, cfg)
        assert np.array_equal(g.color, plain.color) and np.array_equal(g.blend_count, plain.blend_count)
        assert np.array_equal(cache.pixel_offsets, o["offsets"])
        src = np.array([p.source for p in cache.projected])[cache.contribs["proj"]]
        assert np.array_equal(src, o["src"]) and np.array_equal(cache.contribs["alpha"], o["alpha"])
        # the projected list is project_surfel of every projecting surfel, in source order
        ps = [O.project_surfel(sc.surfels[p.source], c, cfg.chi2) for p in cache.projected[:200]]
        for p, q in zip(cache.projected, ps):
            assert np.array_equal(p.h_inv, q["h_inv"]) and p.sort_depth == q["sort_depth"]
        assert cache.grid.rn_total == g.rn_total and sum(len(t) for t in cache.grid.tiles) == g.rn_total
