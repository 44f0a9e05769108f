"""Oracle for the panoptic rows F1/F2, pinned by the reference's own tests:
assign_labels (proj/tests/test_panoptic.cpp:86-183) and the render_panoptic epilogue
(proj/src/metrics.cpp:339-369). CPU only."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2604_10982_b200 import RasterConfig, SceneMap
from paper_2604_10982_b200.panoptic import InstanceQuery, panoptic_epilogue
from tests.helpers import Rng, facing_surfel, front_camera


def surfels_at(centers):
    s = np.zeros((len(centers), 13))
    s[:, 0:3] = centers
    s[:, 3] = 1.0
    s[:, 7:9] = 0.1
    return s


def query(mean, feat, cov):
    return InstanceQuery(feature=np.asarray(feat, float), mean=np.asarray(mean, float), cov=np.asarray(cov, float))


def six_surfels():  # test_panoptic.cpp:87-91
    centers = [(i * 0.3, 0, 0) for i in range(6)]
    f_ins = np.array([[0.1 * i, -0.2] for i in range(6)])
    return surfels_at(centers), f_ins


def test_single_alive_query_claims_everything():  # test_panoptic.cpp:93-100
    s, f = six_surfels()
    dist, arg = O.assign_labels(s, f, [query((0, 0, 0), (1, 1), np.eye(3))])
    assert np.allclose(dist[:, 0], 1.0, rtol=0, atol=1e-12)
    assert np.all(arg == 0)


def test_identical_queries_split_evenly_argmax_lower_index():  # test_panoptic.cpp:102-112
    s, f = six_surfels()
    q = [query((0, 0, 0), (1, 1), np.eye(3)), query((0, 0, 0), (1, 1), np.eye(3))]
    dist, arg = O.assign_labels(s, f, q)
    assert np.allclose(dist, 0.5, rtol=0, atol=1e-12)
    assert np.all(arg == 0)


def attention(q, surf_center, f_ins):  # attention_map (panoptic.cpp:32-34), numpy fp64
    sim = 1.0 / (1.0 + np.exp(-float(np.dot(q.feature, f_ins))))
    cov = 0.5 * (q.cov + q.cov.T)
    d = np.asarray(surf_center) - q.mean
    return sim * np.exp(-0.5 * d @ np.linalg.solve(cov, d))


def test_separated_clusters_match_bruteforce_argmax():  # test_panoptic.cpp:114-149
    rng = Rng(7)
    centers = [np.array([0, 0, 0.]), np.array([5, 0, 0.]), np.array([0, 5, 0.])]
    pts, fs = [], []
    for c in range(3):
        for _ in range(4):
            pts.append(centers[c] + 0.2 * np.array([rng.normal(), rng.normal(), rng.normal()]))
            fs.append([rng.normal(), rng.normal()])
    qs = [query(centers[c], [rng.normal(), rng.normal()], 0.5 * np.eye(3)) for c in range(3)]
    s = surfels_at(pts)
    dist, arg = O.assign_labels(s, np.array(fs), qs)
    for i in range(len(pts)):
        a = [attention(q, pts[i], fs[i]) for q in qs]
        assert arg[i] == int(np.argmax(a))
        assert abs(dist[i].sum() - 1.0) < 1e-8


def test_invariant_under_feature_rotation():  # test_panoptic.cpp:152-183
    rng = Rng(19)
    c_ins = 4
    pts, fs = [], []
    for _ in range(10):
        f = [rng.normal() for _ in range(c_ins)]
        pts.append([rng.normal(), rng.normal(), rng.normal()])
        fs.append(f)
    qs = []
    for _ in range(3):
        f = [rng.normal() for _ in range(c_ins)]
        qs.append(query([rng.normal(), rng.normal(), rng.normal()], f, np.eye(3)))
    s = surfels_at(pts)
    base, barg = O.assign_labels(s, np.array(fs), qs)
    g = np.array([rng.normal() for _ in range(c_ins * c_ins)]).reshape(c_ins, c_ins, order="F")
    rot, _ = np.linalg.qr(g)
    fr = np.array(fs) @ rot.T
    qr = [query(q.mean, rot @ q.feature, q.cov) for q in qs]
    after, aarg = O.assign_labels(s, fr, qr)
    assert np.max(np.abs(base - after)) < 1e-10
    assert np.array_equal(barg, aarg)


def test_dead_queries_get_zero_and_never_win():
    s, f = six_surfels()
    q = [query((0, 0, 0), (1, 1), np.eye(3)), query((0, 0, 0), (5, 5), np.eye(3)), query((1, 0, 0), (1, 0), np.eye(3))]
    q[1].alive = False
    dist, arg = O.assign_labels(s, f, q)
    assert np.all(dist[:, 1] == 0.0)
    assert np.all(arg != 1)
    assert np.allclose(dist.sum(axis=1), 1.0)
    q = [query((0, 0, 0), (1, 1), np.eye(3))]
    q[0].alive = False
    dist, arg = O.assign_labels(s, f, q)
    assert np.all(dist == 0) and np.all(arg == -1)


def test_non_spd_covariance_uses_eps_floor():  # panoptic.cpp:57-61
    s, f = six_surfels()
    singular = np.diag([1.0, 1.0, 0.0])
    dist, arg = O.assign_labels(s, f, [query((0, 0, 0), (1, 1), singular), query((1, 0, 0), (1, 1), np.eye(3))])
    assert np.all(np.isfinite(dist)) and np.allclose(dist.sum(axis=1), 1.0)


def test_panoptic_epilogue_semantics():  # metrics.cpp:349-366
    alpha = np.array([[[0.2], [0.5], [0.9]]])
    arg = np.array([[[3], [1], [-1]]], np.int32)
    sem = np.array([[[1.0, 2.0], [3.0, 3.0], [0.0, -1.0]]])
    pr = panoptic_epilogue(alpha, arg, sem, [10, 11])
    assert pr.ids[..., 0].tolist() == [[-1, 1, -1]]
    assert pr.classes[..., 0].tolist() == [[-1, 11, -1]]
    assert pr.sem_classes[..., 0].tolist() == [[-1, 0, 0]]  # ties -> first index


def test_render_panoptic_oracle_small():
    cam = front_camera(32, 32)
    rows = [facing_surfel((x, 0, 2.0 + 0.1 * i), 0.2, 0.2, 0.9, (0.5, 0.5, 0.5)) for i, x in enumerate((-0.3, 0.0, 0.3))]
    sc = SceneMap(np.array(rows), np.array([[1.0, 0.0], [0.0, 1.0], [0.5, 0.4]]))
    f_ins = np.array([[1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    qs = [query((-0.3, 0, 2), (2, 0), 0.05 * np.eye(3)), query((0.3, 0, 2.2), (0, 2), 0.05 * np.eye(3))]
    qs[0].class_id, qs[1].class_id = 4, 7
    out = O.render_panoptic(sc, f_ins, qs, cam, RasterConfig())
    ids = out["ids"][..., 0]
    assert set(np.unique(ids)) <= {-1, 0, 1}
    assert np.all((out["classes"][..., 0] == -1) == (ids == -1))
    assert np.all(out["classes"][..., 0][ids == 0] == 4) and np.all(out["classes"][..., 0][ids == 1] == 7)
    assert np.any(ids == 0) and np.any(ids == 1)
