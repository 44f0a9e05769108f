"""Oracle for the render backward: the blending backward of
pipeline.cpp:347-460 and project_surfel_backward (raster.cpp:179-203), pinned the way the
reference pins it (test_gradients.cpp:150-177): central finite differences of
L = <g_color, colour> + <g_sem, sem_feat> + <g_ins, ins_dist> on the oracle forward.
CPU only."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2604_10982_b200 import Blending, RasterConfig, SceneMap
from tests.helpers import front_camera


def scene_case(seed, n=8, c_sem=3, n_q=2):
    rng = np.random.default_rng(seed)
    s = np.zeros((n, 13))
    s[:, 0] = rng.uniform(-0.25, 0.25, n)
    s[:, 1] = rng.uniform(-0.25, 0.25, n)
    s[:, 2] = rng.uniform(1.8, 2.6, n)
    q = rng.normal(size=(n, 4)) * 0.25 + np.array([1.0, 0, 0, 0])
    s[:, 3:7] = q / np.linalg.norm(q, axis=1, keepdims=True)
    s[:, 7] = rng.uniform(0.08, 0.2, n)
    s[:, 8] = rng.uniform(0.05, 0.15, n)
    s[:, 9] = rng.uniform(0.3, 0.8, n)
    s[:, 10:13] = rng.uniform(0.1, 0.9, (n, 3))
    f = rng.normal(size=(n, c_sem))
    lab = rng.dirichlet(np.ones(n_q), size=n)
    return SceneMap(s, f), lab


def loss(scene, lab, cam, cfg, gc, gs, gi):
    o = O.render(scene, lab, cam, cfg)
    return float(np.sum(gc * o["color"]) + np.sum(gs * o["sem_feat"]) + np.sum(gi * o["ins_dist"]))


PARAMS = [("center", 0, 3), ("rotation", 3, 4), ("scales", 7, 2), ("opacity", 9, 1), ("color", 10, 3)]


@pytest.mark.parametrize("blending,k", [(Blending.Full, 16), (Blending.TopK, 2)])
def test_backward_matches_finite_differences(blending, k):
    scene, lab = scene_case(5)
    cam = front_camera(32, 32, 60.0)
    cfg = RasterConfig(blending=blending, top_k=k)
    rng = np.random.default_rng(9)
    gc = rng.normal(size=(32, 32, 3))
    gs = rng.normal(size=(32, 32, scene.c_sem()))
    gi = rng.normal(size=(32, 32, lab.shape[1]))
    g = O.render_backward(scene, lab, cam, cfg, gc, gs, gi)
    checked, worst = 0, 0.0
    for name, col, width in PARAMS:
        for i in range(len(scene)):
            for c in range(width):
                for arr, j in ((scene.surfels, col + c),):
                    eps = 1e-6
                    base = arr[i, j]
                    arr[i, j] = base + eps
                    lp = loss(scene, lab, cam, cfg, gc, gs, gi)
                    arr[i, j] = base - eps
                    lm = loss(scene, lab, cam, cfg, gc, gs, gi)
                    arr[i, j] = base
                    num = (lp - lm) / (2 * eps)
                    ana = g[name][i, c] if g[name].ndim == 2 else g[name][i]
                    err = abs(num - ana) / max(abs(num), abs(ana), 1e-3)
                    worst = max(worst, err)
                    checked += 1
    assert checked == len(scene) * 13
    assert worst < 1e-4, worst
    # features and labels enter linearly: their FD is exact in closed form
    for name, arr in (("f_sem", scene.f_sem), ("labels", lab)):
        for i in range(len(scene)):
            for c in range(arr.shape[1]):
                base = arr[i, c]
                arr[i, c] = base + 1e-3
                lp = loss(scene, lab, cam, cfg, gc, gs, gi)
                arr[i, c] = base - 1e-3
                lm = loss(scene, lab, cam, cfg, gc, gs, gi)
                arr[i, c] = base
                num = (lp - lm) / 2e-3
                assert abs(num - g[name][i, c]) <= 1e-7 * max(1.0, abs(num)), (name, i, c)


def test_zero_upstream_gives_zero_gradients():  # test_gradients.cpp:87-115
    scene, lab = scene_case(3)
    cam = front_camera(32, 32, 60.0)
    g = O.render_backward(scene, lab, cam, RasterConfig())
    assert all(np.all(v == 0) for v in g.values())


def test_single_surfel_colour_derivative():  # test_gradients.cpp:117-148: dL/dc = sum of weights
    s = np.zeros((1, 13))
    s[0, 2] = 2.0
    s[0, 3] = 1.0
    s[0, 7:9] = 0.1
    s[0, 9] = 0.5
    s[0, 10:13] = 0.5
    scene = SceneMap(s)
    cam = front_camera(16, 16, 60.0)
    gc = np.zeros((16, 16, 3))
    gc[..., 0] = 1.0
    g = O.render_backward(scene, None, cam, RasterConfig(), gc)
    o = O.render(scene, None, cam, RasterConfig())
    # colour_r = w * c_r per pixel with a single contributor: dL/dc_r = sum_px w = sum_px alpha_acc
    assert abs(g["color"][0, 0] - o["alpha_acc"].sum()) < 1e-12
    assert g["color"][0, 1] == 0 and g["color"][0, 2] == 0
