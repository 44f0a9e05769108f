"""Pins the CPU oracle (oracle/oracle.cpp) and the host workload generator to the REFERENCE'S
OWN CODE: proj/src/{raster,math_util,core_types,synthetic}.cpp compiled unchanged into
oracle/_ref (oracle/ref/Makefile, against the minimal Eigen stand-in oracle/eigen_min).

Bit-exact, every fp64 / int32 plane of render_into (raster.cpp:273-511), the tile lists of
bin_circle / bin_aabb (raster.cpp:51-90,144-152), the bench_render counters
(raster.cpp:513-573), the stage functions (project_surfel, evaluate_alpha, topk_select), the
street-scene generator (synthetic.cpp:236-312) and Camera::look_at (core_types.cpp:40-60).
Non-identity camera poses (the C5 trajectory, an arbitrary Camera::make pose) exercise the
camera transform products (raster.cpp:96-101, core_types.hpp:51-52) bit for bit. The panoptic
rows (panoptic.cpp assign_labels, metrics.cpp render_panoptic) and the backward row
(raster.cpp project_surfel_backward, pipeline.cpp pipeline_backward) are pinned the same way.

The oracle's parity build uses psm_exp (the GPU's exp); the libm build uses glibc exp like
the reference. Both must match the reference exactly: psm_exp restates glibc's FMA exp.
"""
import math

import numpy as np
import pytest

from oracle import pyoracle as O
from oracle import pyref as R
from paper_2604_10982_b200 import (Binning, Blending, Camera, RasterConfig, SceneMap, StreetSpec, density_scale,
                                   make_street_scene, trajectory_cameras)
from tests.helpers import Rng

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built (needs /root/reference)")

PLANES = ("color", "depth", "normal", "sem_feat", "ins_dist", "ins_argmax", "alpha_acc", "blend_count")


def assert_oracle_is_reference(rs: R.RefScene, scene, labels, cam, cfg, libm_too=True):
    r = rs.render(cam, cfg)
    for libm in ((False, True) if libm_too else (False,)):
        o = O.render(scene, labels, cam, cfg, libm=libm)
        for k in PLANES:
            assert r[k].shape == o[k].shape, k
            assert np.array_equal(r[k], o[k]), (k, "libm" if libm else "psm_exp",
                                                 int(np.count_nonzero(r[k] != o[k])))
        assert r["blended_total"] == o["counters"]["blended_total"]
    return r


@pytest.fixture(scope="module")
def c0():
    """C0: the reference-standard street scene (12k surfels, 256x192, C_sem 32, 256 labels, seed 7)."""
    s, f, lab, fi, camc = R.make_street_scene()
    return s, f, lab, fi, Camera.from_c(camc), R.RefScene(s, f, lab)


def test_street_scene_generator_is_the_reference(c0):
    s, f, lab, fi, cam, _ = c0
    sc, lab2, cam2 = make_street_scene(StreetSpec())
    assert np.array_equal(sc.surfels, s) and np.array_equal(sc.f_sem, f) and np.array_equal(lab2, lab)
    assert bytes(cam2.to_c()) == bytes(cam.to_c())
    from paper_2604_10982_b200 import street_f_ins
    assert np.array_equal(street_f_ins(StreetSpec()), fi)


def test_street_scene_generator_c3_shape_and_scale_mult():
    """C3-shaped spec (1280x720, C_sem 64). scale_mult multiplies s1 right after it is
    drawn: every other draw, and s1 itself up to that product, is the reference's."""
    kw = dict(n_surfels=20000, image_w=1280, image_h=720, c_sem=64, n_instances=32)
    s, f, lab, fi, camc = R.make_street_scene(**kw)
    sc, lab2, cam2 = make_street_scene(StreetSpec(**kw))
    assert np.array_equal(sc.surfels, s) and np.array_equal(sc.f_sem, f) and np.array_equal(lab2, lab)
    assert bytes(cam2.to_c()) == bytes(camc)
    k = density_scale(20000, 1280, 720)
    sk, _, _ = make_street_scene(StreetSpec(scale_mult=k, **kw), with_labels=False)
    other = [c for c in range(13) if c not in (7, 8)]
    assert np.array_equal(sk.surfels[:, other], s[:, other]) and np.array_equal(sk.f_sem, f)
    assert np.array_equal(sk.surfels[:, 7], s[:, 7] * k)
    np.testing.assert_allclose(sk.surfels[:, 8], s[:, 8] * k, rtol=1e-14)


def test_oracle_generator_is_the_reference():
    """The oracle's own generator (used by bench.py's reference arm) equals the reference's."""
    kw = dict(n_surfels=5000, image_w=320, image_h=180, c_sem=16, n_instances=8)
    s, f, lab, _, camc = R.make_street_scene(**kw)
    so, fo, labo, camo = O.make_street_scene(StreetSpec(**kw), with_labels=True)
    assert np.array_equal(so, s) and np.array_equal(fo, f) and np.array_equal(labo, lab)
    assert bytes(camo) == bytes(camc)


def test_look_at_is_the_reference():
    import ctypes as C
    from paper_2604_10982_b200 import _abi as A
    for i in (0, 1, 37, 64, 128, 200, 255):
        a = 2.0 * math.pi * i / 256
        eye = (0.8 * math.sin(a), 0.2 * math.sin(2.0 * a), 0.05 * i)
        th = 0.15 * math.sin(a)
        tgt = (eye[0] + 20.0 * math.sin(th), eye[1], eye[2] + 20.0 * math.cos(th))
        ours = trajectory_cameras(256, 1920, 1080, first=i, count=1)[0]
        rc = A.psm_camera()
        arr = lambda v: (C.c_double * 3)(*v)
        assert R.load().ref_camera_look_at(arr(eye), arr(tgt), arr((0.0, -1.0, 0.0)), 0.8 * 1920, 0.8 * 1920, 1920,
                                           1080, 0.1, 200.0, C.byref(rc)) == 0
        assert bytes(ours.to_c()) == bytes(rc), i


@pytest.mark.parametrize("binning", [Binning.Circle, Binning.Aabb])
@pytest.mark.parametrize("blending,k", [(Blending.Full, 16), (Blending.TopK, 16), (Blending.TopK, 8)])
def test_oracle_is_reference_c0(c0, binning, blending, k):
    s, f, lab, _, cam, rs = c0
    assert_oracle_is_reference(rs, SceneMap(s, f), lab, cam, RasterConfig(binning=binning, blending=blending, top_k=k))


def test_oracle_is_reference_config_variants(c0):
    s, f, lab, _, cam, rs = c0
    sc = SceneMap(s, f)
    for cfg in (RasterConfig(support_cutoff=False), RasterConfig(render_depth_normal=False, blending=Blending.TopK),
                RasterConfig(background=(0.2, 0.4, 0.6), t_min=1e-2, alpha_min=0.05, chi2=4.0),
                RasterConfig(blending=Blending.TopK, top_k=1), RasterConfig(blending=Blending.TopK, top_k=0),
                RasterConfig(tile_size=8), RasterConfig(tile_size=32, blending=Blending.TopK, top_k=5)):
        assert_oracle_is_reference(rs, sc, lab, cam, cfg, libm_too=False)


def test_bin_lists_are_reference(c0):
    s, f, lab, _, cam, rs = c0
    for cams in ([cam], trajectory_cameras(256, 256, 192, first=3, count=1)):
        for binning in (Binning.Circle, Binning.Aabb):
            cfg = RasterConfig(binning=binning)
            r = rs.bin(cams[0], cfg, binning)
            o = O.bin_surfels(s, cams[0], cfg, binning)
            assert r["rn_total"] == o["rn_total"] and r["n_proj"] == o["n_proj"]
            assert r["rn_per_tile"] == o["rn_per_tile"]
            assert all(np.array_equal(a, b) for a, b in zip(r["tiles"], o["tiles"]))


def test_bench_render_counters_are_reference(c0):
    """bench_render rows (raster.cpp:513-573): rn_total, rn_per_tile, blended_total identical."""
    s, f, lab, _, cam, rs = c0
    rows = rs.bench_render(cam, 1, RasterConfig(top_k=16))
    for i, (binning, blending) in enumerate([(Binning.Circle, Blending.Full), (Binning.Aabb, Blending.Full),
                                             (Binning.Circle, Blending.TopK), (Binning.Aabb, Blending.TopK)]):
        o = O.render(SceneMap(s, f), lab, cam, RasterConfig(binning=binning, blending=blending, top_k=16),
                     planes=False)["counters"]
        assert rows[i, 2] == o["rn_total"] and rows[i, 3] == o["rn_per_tile"] and rows[i, 4] == o["blended_total"]
    assert rows[2, 4] == rows[3, 4]  # test_raster.cpp:372-390


def _pose_cameras(w, h):
    """Non-identity poses: C5 trajectory views and an arbitrary Camera::make pose with translation."""
    cams = trajectory_cameras(256, w, h, first=0, count=256)
    picks = [cams[i] for i in (5, 64, 131, 250)]
    # a yaw + roll about the street camera (keeps the scene in view), translated, off-centre principal point
    a, b = 0.07, 0.05
    yaw = np.array([[math.cos(a), 0, math.sin(a)], [0, 1, 0], [-math.sin(a), 0, math.cos(a)]])
    roll = np.array([[math.cos(b), -math.sin(b), 0], [math.sin(b), math.cos(b), 0], [0, 0, 1]])
    tilt = roll @ yaw
    picks.append(Camera.make(tilt, np.array([0.3, -0.2, 1.7]), 0.75 * w, 0.8 * w, 0.47 * w, 0.53 * h, w, h, 0.1,
                             200.0))
    return picks


@pytest.mark.parametrize("blending,k", [(Blending.TopK, 16), (Blending.Full, 16)])
def test_oracle_is_reference_non_identity_poses(c0, blending, k):
    s, f, lab, _, cam, rs = c0
    for pc in _pose_cameras(256, 192):
        assert_oracle_is_reference(rs, SceneMap(s, f), lab, pc, RasterConfig(blending=blending, top_k=k),
                                   libm_too=False)


def test_oracle_is_reference_100k_1280x720():
    """>= 100k surfels at 1280x720 (C3 shape, density-normalised, 64-d features, K = 8), the street
    camera and one trajectory pose."""
    n, w, h = 100_000, 1280, 720
    sc, _, cam = make_street_scene(StreetSpec(n_surfels=n, image_w=w, image_h=h, c_sem=64,
                                              scale_mult=density_scale(n, w, h)), with_labels=False)
    rs = R.RefScene(sc.surfels, sc.f_sem, None)
    cfg = RasterConfig(binning=Binning.Aabb, blending=Blending.TopK, top_k=8)
    for c in (cam, trajectory_cameras(256, w, h, first=77, count=1)[0]):
        assert_oracle_is_reference(rs, sc, None, c, cfg, libm_too=False)
    rs.close()


def test_stage_functions_are_reference():
    """project_surfel, evaluate_alpha (raster.cpp:94-177) and topk_select (raster.cpp:225-251)."""
    rng = Rng(5)
    cams = _pose_cameras(320, 240)
    cfg = RasterConfig()
    for i in range(400):
        c = cams[i % len(cams)]
        q = rng.unit_quaternion()
        s13 = np.array([rng.uniform(-3, 3), rng.uniform(-2, 2), rng.uniform(-1, 25), *q, rng.uniform(0.01, 1.5),
                        rng.uniform(0.01, 0.4), rng.uniform(0.1, 1), 0.5, 0.5, 0.5])
        pr, po = R.project_surfel(s13, c, cfg), O.project_surfel(s13, c, cfg.chi2)
        assert (pr is None) == (po is None)
        if pr is not None:
            for k in pr:
                assert np.array_equal(np.asarray(pr[k]), np.asarray(po[k])), k
            for _ in range(4):
                px, py = pr["center"] + np.array([rng.uniform(-6, 6), rng.uniform(-6, 6)])
                px, py = math.floor(px) + 0.5, math.floor(py) + 0.5
                ar, ao = R.evaluate_alpha(s13, c, px, py, cfg), O.evaluate_alpha(s13, c, px, py, cfg)
                assert ar == ao
    for m in (1, 5, 9, 40):
        for k in (1, 4, 8, 16):
            w = np.array([rng.uniform() for _ in range(m)])
            w[: m // 3] = w[0]  # ties broken by proj ascending
            p = np.array([int(rng.uniform_int(1000)) for _ in range(m)], np.int32)
            assert np.array_equal(R.topk_select(w, p, k), O.topk_select(w, p, k))


# ---- panoptic rows (F1 assign_labels, F2 render_panoptic): panoptic.cpp / metrics.cpp compiled in _ref
def _panoptic_street(n=12000, w=256, h=192, c_sem=32, n_queries=24):
    from paper_2604_10982_b200 import street_f_ins, street_queries
    spec = StreetSpec(n_surfels=n, image_w=w, image_h=h, c_sem=c_sem, seed=7)
    sc, _, cam = make_street_scene(spec, with_labels=False)
    qs = street_queries(n_queries, c_ins=8)
    qs[3].alive = False
    qs[11].alive = False
    return SceneMap(sc.surfels, sc.f_sem, street_f_ins(spec), qs), cam


def test_assign_labels_is_reference():
    """The oracle's assign_labels (psm_panoptic.h, shared with the GPU) equals the reference's bit for bit:
    Eigen's dynamic dot order, LLT and its triangular solve as modelled by oracle/eigen_min."""
    sc, _ = _panoptic_street()
    rd, ra = R.assign_labels(sc.surfels, sc.f_ins, sc.queries)
    od, oa = O.assign_labels(sc.surfels, sc.f_ins, sc.queries)
    assert np.array_equal(ra, oa)
    assert np.array_equal(rd.view(np.uint64), od.view(np.uint64))
    # odd feature widths and non-trivial covariances (the LLT retry, the dot's tail)
    from paper_2604_10982_b200 import InstanceQuery
    rng = np.random.default_rng(1)
    for c_ins in (1, 3, 5, 8, 13, 16):
        f = rng.standard_normal((500, c_ins))
        qs = []
        for i in range(9):
            a = rng.standard_normal((3, 3))
            cov = a @ a.T + (0.0 if i == 4 else 0.1) * np.eye(3)
            if i == 6:
                cov = np.diag([1.0, 1.0, 0.0])  # not positive definite: the eps retry
            qs.append(InstanceQuery(rng.standard_normal(c_ins), rng.uniform(-2, 2, 3), cov, alive=i != 2))
        s = np.zeros((500, 13))
        s[:, :3] = rng.uniform(-3, 3, (500, 3))
        s[:, 3] = 1.0
        rd, ra = R.assign_labels(s, f, qs)
        od, oa = O.assign_labels(s, f, qs)
        assert np.array_equal(ra, oa) and np.array_equal(rd.view(np.uint64), od.view(np.uint64)), c_ins


@pytest.mark.parametrize("blending,k", [(Blending.TopK, 16), (Blending.Full, 16), (Blending.TopK, 8)])
def test_render_panoptic_is_reference(blending, k):
    sc, cam = _panoptic_street()
    cfg = RasterConfig(binning=Binning.Aabb, blending=blending, top_k=k)
    r = R.render_panoptic(sc, cam, cfg)
    o = O.render_panoptic(sc, sc.f_ins, sc.queries, cam, cfg)
    for key in ("ids", "classes", "sem_classes"):
        assert np.array_equal(r[key], o[key]), key


# ---- backward row (F4): raster.cpp project_surfel_backward and pipeline.cpp pipeline_backward in _ref
def test_project_surfel_backward_is_reference():
    """project_surfel_backward (raster.cpp:179-203) vs psm_geom_backward (the oracle's and the GPU's),
    bit for bit, under non-identity poses."""
    rng = Rng(11)
    cams = _pose_cameras(320, 240)
    cfg = RasterConfig()
    projected = 0
    for i in range(300):
        c = cams[i % len(cams)]
        q = rng.unit_quaternion()
        s13 = np.array([rng.uniform(-3, 3), rng.uniform(-2, 2), rng.uniform(-1, 25), *q, rng.uniform(0.01, 1.5),
                        rng.uniform(0.01, 0.4), rng.uniform(0.1, 1), 0.5, 0.5, 0.5])
        g = np.array([rng.uniform(-1, 1) for _ in range(9)]).reshape(3, 3)
        r, o = R.project_surfel_backward(s13, c, cfg, g), O.project_surfel_backward(s13, c, g, cfg.chi2)
        assert (r is None) == (o is None)
        if r is None:
            continue
        projected += 1
        for k in r:
            assert np.array_equal(r[k], o[k]), (i, k)
    assert projected > 150


def sem_ce_plane_grad(sem_feat, sem_gt, l_sem):
    """d L_sem / d sem_feat of the clamped cross-entropy as pipeline_backward forms it
    (pipeline.cpp:270-295); math.exp is the C library's exp, like the reference's std::exp."""
    h, w, c_sem = sem_feat.shape
    g = np.zeros_like(sem_feat)
    labeled = int((sem_gt >= 0).sum())
    if labeled == 0:
        return g
    scale = l_sem / labeled
    for y in range(h):
        for x in range(w):
            cls = int(sem_gt[y, x])
            if cls < 0:
                continue
            f = sem_feat[y, x]
            m = f[0]
            for i in range(1, c_sem):
                m = max(m, f[i])
            den = 0.0
            for i in range(c_sem):
                den += math.exp(f[i] - m)
            p_cls = math.exp(f[cls] - m) / den
            if p_cls < 1e-7 or p_cls > 1.0 - 1e-7:
                continue
            for i in range(c_sem):
                g[y, x, i] = scale * (math.exp(f[i] - m) / den - (1.0 if i == cls else 0.0))
    return g


SMOOTH = RasterConfig(alpha_min=0.0, t_min=0.0, support_cutoff=False, chi2=1e8, blending=Blending.Full)  # pipeline.cpp:56-64


@pytest.mark.parametrize("case", ["topk4", "full", "smooth"])
def test_pipeline_backward_is_reference(case):
    """The oracle's blending backward + geometry chain (oracle_render_backward) against the reference's own
    pipeline_backward (pipeline.cpp:253-600) on a query-free scene without a SOGMM model and l_iso = 0, so
    that every surfel gradient comes from the render: the upstream colour plane is the reference's own
    loss_rgb_backward, the semantic plane its clamped cross-entropy (restated above). Bit for bit: the
    oracle sums in the reference's 16 pixel chunks, merged in order."""
    sc, _, cam = make_street_scene(StreetSpec(n_surfels=3000, image_w=96, image_h=64, c_sem=6), with_labels=False)
    rs = R.RefScene(sc.surfels, sc.f_sem, None)
    rng = np.random.default_rng(3)
    rgb = rng.uniform(0, 1, (64, 96, 3))
    sem = rng.integers(-1, 6, (64, 96)).astype(np.int32)
    cfg = {"topk4": RasterConfig(blending=Blending.TopK, top_k=4), "full": RasterConfig(),
           "smooth": SMOOTH}[case]
    pose = _pose_cameras(96, 64)[4]
    for c in (cam, pose):
        r = rs.pipeline_backward(c, cfg, rgb, sem, l_sem=0.5, l_iso=0.0, smooth=case == "smooth")
        g_sem = sem_ce_plane_grad(rs.render(c, cfg)["sem_feat"], sem, 0.5)
        o = O.render_backward(sc, None, c, cfg, g_color=r["g_color_plane"], g_sem=g_sem)
        for k in ("opacity", "color", "f_sem", "center", "rotation", "scales"):
            assert np.count_nonzero(r[k]) > 0, k
            assert np.array_equal(r[k], o[k]), (case, k, float(np.max(np.abs(r[k] - o[k]))))
    rs.close()
