"""Pins the CPU oracle to the reference: every known-answer test of
proj/tests/test_raster.cpp and acceptance criteria 1-3 (proj/tests/acceptance.cpp:44-167),
ported case by case, plus the oracle's own pins (psm_exp vs glibc exp, the
Ellipse binning extension's conservativeness and output identity).

CPU only (no GPU); these decide whether the oracle may be trusted as the parity checker.
"""
import math
import time

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2604_10982_b200 import Binning, Blending, RasterConfig, SceneMap, StreetSpec, make_street_scene
from tests.helpers import Rng, facing_surfel, front_camera, scene_of


def approx(a, b, eps):  # doctest::Approx(b).epsilon(eps)
    return abs(a - b) <= eps * (1.0 + max(abs(a), abs(b)))


# ------------------------------------------------------------ test_raster.cpp:41-54
def test_projection_pinhole_scaling():
    cam = front_camera()
    p = O.project_surfel(facing_surfel((0, 0, 2), 0.1, 0.1, 1.0, (1, 0, 0)), cam)
    assert p is not None
    # sigma_px = s f / z = 0.1 * 100 / 2 = 5 -> sigma' = diag(25, 25)
    assert approx(p["sigma"][0, 0], 25.0, 1e-9)
    assert approx(p["sigma"][1, 1], 25.0, 1e-9)
    assert abs(p["sigma"][0, 1]) < 1e-9
    assert approx(p["sort_depth"], 2.0, 1e-12)
    assert approx(p["center"][0], cam.cx, 1e-12)
    assert approx(p["center"][1], cam.cy, 1e-12)


# ------------------------------------------------------------ test_raster.cpp:56-68
def test_projection_culls_behind_and_grazing():
    cam = front_camera()
    assert O.project_surfel(facing_surfel((0, 0, -2), 0.1, 0.1, 1, (1, 0, 0)), cam) is None
    c, sn = math.cos(math.pi / 4), math.sin(math.pi / 4)
    graze = facing_surfel((0, 0, 2), 0.1, 0.1, 1, (1, 0, 0), quat=(c, sn, 0, 0))
    assert O.project_surfel(graze, cam) is None


# ------------------------------------------------------------ test_raster.cpp:70-103
def test_edge_on_surfel_homography_matches_ray_plane():
    cam = front_camera()
    cfg = RasterConfig(support_cutoff=False)
    ang = 88.0 * math.pi / 180.0
    s = facing_surfel((0.3, 0, 2), 0.4, 0.4, 1.0, (1, 0, 0), quat=(math.cos(ang / 2), 0, math.sin(ang / 2), 0))
    p = O.project_surfel(s, cam)
    assert p is not None
    sg = p["sigma"]
    lmin = 0.5 * (np.trace(sg) - math.sqrt((sg[0, 0] - sg[1, 1]) ** 2 + 4 * sg[0, 1] ** 2))
    lmax = np.trace(sg) - lmin
    assert lmin / lmax < 0.05
    px, py = p["center"][0] + 1.0, p["center"][1]
    smp = O.evaluate_alpha(s, cam, px, py, cfg)
    assert smp["inside"] and math.isfinite(smp["u"]) and math.isfinite(smp["v"])
    ray = np.array([(px - cam.cx) / cam.fx, (py - cam.cy) / cam.fy, 1.0])
    w, x, y, z = s[3:7]
    r = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                  [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                  [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
    n = r[:, 2]
    t = n.dot(s[:3]) / n.dot(ray)
    hit = t * ray
    u_direct = (hit - s[:3]).dot(r[:, 0]) / s[7]
    v_direct = (hit - s[:3]).dot(r[:, 1]) / s[8]
    assert approx(smp["u"], u_direct, 1e-8)
    assert approx(smp["v"], v_direct, 1e-8)
    assert approx(1.0 / smp["w2"], t, 1e-8)


# ------------------------------------------------------------ test_raster.cpp:105-125
def test_evaluate_alpha_closed_forms():
    cam = front_camera()
    cfg = RasterConfig()
    s = facing_surfel((0, 0, 2), 0.1, 0.1, 0.8, (1, 0, 0))
    assert approx(O.evaluate_alpha(s, cam, cam.cx, cam.cy, cfg)["alpha"], 0.8, 1e-12)
    px, py = cam.cx + 5.0, cam.cy + 5.0
    assert approx(O.evaluate_alpha(s, cam, px, py, cfg)["alpha"], 0.8 * math.exp(-1.0), 1e-9)
    wide = RasterConfig(chi2=100.0)
    assert O.evaluate_alpha(s, cam, cam.cx + 20.0, cam.cy + 20.0, wide)["alpha"] == 0.0


# ------------------------------------------------------------ test_raster.cpp:127-147
def test_binning_isotropic_footprints_identical():
    cam = front_camera()
    cfg = RasterConfig()
    rng = Rng(5)
    rows = []
    for _ in range(40):
        c = (rng.uniform(-0.5, 0.5), rng.uniform(-0.5, 0.5), rng.uniform(1.5, 4.0))
        rows.append(facing_surfel(c, 0.08, 0.08, 0.9, (1, 1, 1)))
    a = O.bin_surfels(rows, cam, cfg, 0)
    b = O.bin_surfels(rows, cam, cfg, 1)
    for ta, tb in zip(a["tiles"], b["tiles"]):
        assert np.array_equal(ta, tb)
    assert a["rn_total"] == b["rn_total"]


# ------------------------------------------------------------ test_raster.cpp:149-170
def test_binning_elongated_aabb_strictly_fewer():
    cam = front_camera(128, 128)
    cfg = RasterConfig()
    s = facing_surfel((0, 0, 2), 0.4, 0.02, 0.9, (1, 1, 1))
    p = O.project_surfel(s, cam)
    assert approx(p["sigma"][0, 0], 400.0, 1e-9)
    assert approx(p["sigma"][1, 1], 1.0, 1e-9)
    a = O.bin_surfels([s], cam, cfg, 0)
    b = O.bin_surfels([s], cam, cfg, 1)
    assert b["rn_total"] == 8 * 2  # aabb: x tiles 0..7, y tiles 3..4
    assert a["rn_total"] > b["rn_total"]
    assert a["rn_total"] == 64
    e = O.bin_surfels([s], cam, cfg, 2)  # the exact ellipse test never keeps more than the AABB
    assert e["rn_total"] <= b["rn_total"]


# ------------------------------------------------------------ test_raster.cpp:172-199
def _random_surfels(seed, n, lo=0.02, hi=0.5):
    rng = Rng(seed)
    rows = []
    for _ in range(n):
        c = (rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(1, 6))
        s1, s2 = rng.uniform(lo, hi), rng.uniform(lo, hi)
        q = rng.unit_quaternion()
        rows.append(facing_surfel(c, s1, s2, 0.9, (1, 1, 1), quat=q))
    return rows


def test_aabb_never_assigns_more_tiles_than_circle():
    cam = front_camera(128, 96)
    cfg = RasterConfig()
    rows = _random_surfels(9, 200)
    a = O.bin_surfels(rows, cam, cfg, 0)
    b = O.bin_surfels(rows, cam, cfg, 1)
    e = O.bin_surfels(rows, cam, cfg, 2)
    assert np.all(b["per_surfel"] <= a["per_surfel"])
    assert np.all(e["per_surfel"] <= b["per_surfel"])
    assert b["rn_total"] <= a["rn_total"]


# ------------------------------------------------------------ test_raster.cpp:201-216
def test_render_single_opaque_surfel():
    cam = front_camera()
    sc = scene_of([facing_surfel((0, 0, 2), 0.2, 0.2, 1.0, (0.3, 0.6, 0.9))])
    out = O.render(sc, None, cam, RasterConfig(background=(0.1, 0.1, 0.1)))
    x, y = int(cam.cx), int(cam.cy)
    assert approx(out["color"][y, x, 0], 0.3, 1e-12)
    assert approx(out["color"][y, x, 1], 0.6, 1e-12)
    assert approx(out["color"][y, x, 2], 0.9, 1e-12)
    assert approx(out["alpha_acc"][y, x, 0], 1.0, 1e-12)
    assert approx(out["depth"][y, x, 0], 2.0, 1e-9)
    assert approx(out["depth"][y, x, 1], 2.0, 1e-9)


# ------------------------------------------------------------ test_raster.cpp:218-231
def test_render_two_surfel_alpha_arithmetic():
    cam = front_camera()
    sc = scene_of([facing_surfel((0, 0, 2), 0.2, 0.2, 0.5, (1, 0, 0)),
                   facing_surfel((0, 0, 3), 0.3, 0.3, 1.0, (0, 1, 0))])
    out = O.render(sc, None, cam, RasterConfig())
    x, y = int(cam.cx), int(cam.cy)
    assert approx(out["color"][y, x, 0], 0.5, 1e-12)
    assert approx(out["color"][y, x, 1], 0.5, 1e-12)
    assert approx(out["color"][y, x, 2], 0.0, 1e-12)


# ------------------------------------------------------------ test_raster.cpp:233-248
def test_render_empty_scene_background():
    cam = front_camera(16, 16)
    out = O.render(SceneMap(np.zeros((0, 13))), None, cam, RasterConfig(background=(0.25, 0.5, 0.75)))
    assert np.all(out["color"][..., 0] == 0.25)
    assert np.all(out["color"][..., 1] == 0.5)
    assert np.all(out["color"][..., 2] == 0.75)
    assert np.all(out["alpha_acc"] == 0.0)
    assert np.all(out["ins_argmax"] == -1)


def _street(n, w, h, c_sem, **kw):
    return make_street_scene(StreetSpec(n_surfels=n, image_w=w, image_h=h, c_sem=c_sem, **kw))


# ------------------------------------------------------------ test_raster.cpp:250-267
def test_binning_soundness_circle_vs_aabb_color():
    sc, labels, cam = _street(400, 96, 64, 4)
    a = O.render(sc, labels, cam, RasterConfig(binning=Binning.Circle))
    b = O.render(sc, labels, cam, RasterConfig(binning=Binning.Aabb))
    assert np.max(np.abs(a["color"] - b["color"])) < 1e-6


# ------------------------------------------------------------ test_raster.cpp:269-298
def test_depth_order_permutation_bit_identical():
    sc, labels, cam = _street(200, 64, 48, 3)
    n = len(sc)
    perm = list(range(n))
    rng = Rng(13)
    for i in range(n - 1, 0, -1):
        j = rng.uniform_int(i + 1)
        perm[i], perm[j] = perm[j], perm[i]
    perm = np.array(perm)
    sh = SceneMap(sc.surfels[perm], sc.f_sem[perm])
    cfg = RasterConfig()
    a = O.render(sc, labels, cam, cfg)
    b = O.render(sh, labels[perm], cam, cfg)
    for k in ("color", "sem_feat", "ins_dist", "depth"):
        assert np.array_equal(a[k], b[k]), k


# ------------------------------------------------------------ test_raster.cpp:300-313
def test_transmittance_invariant():
    sc, labels, cam = _street(300, 64, 48, 2)
    out = O.render(sc, labels, cam, RasterConfig())
    assert np.all(out["alpha_acc"] >= 0.0)
    assert np.all(out["alpha_acc"] <= 1.0 + 1e-12)


# ------------------------------------------------------------ test_raster.cpp:315-370
def _stacked_scene():
    rng = Rng(31)
    n = 50
    rows, fs = [], []
    for i in range(n):
        # facing_surfel(Vec3(u, u, 1.5 + 0.05 i), 0.3, 0.3, u(0.03, 0.12), ...): the draw order of the
        # reference's unsequenced arguments is compiler-defined; the tail-bound property holds for any
        c = (rng.uniform(-0.02, 0.02), rng.uniform(-0.02, 0.02), 1.5 + 0.05 * i)
        o = rng.uniform(0.03, 0.12)
        rows.append(facing_surfel(c, 0.3, 0.3, o, (0.5, 0.5, 0.5)))
        fs.append([rng.uniform(-1, 1), rng.uniform(-1, 1)])
    labels = np.full((n, 4), 0.25)
    return SceneMap(np.array(rows), np.array(fs)), labels


def _tail_bound_holds(full_cache, sel_sem, full_sem, f_sem, k, slack):
    offs, src, alpha = full_cache["offsets"], full_cache["src"], full_cache["alpha"]
    h, w = sel_sem.shape[:2]
    for p in range(w * h):
        a = alpha[offs[p]:offs[p + 1]]
        if len(a) == 0:
            continue
        t = np.concatenate([[1.0], np.cumprod(1.0 - a)[:-1]])
        wts = a * t
        max_f = np.max(np.abs(f_sem[src[offs[p]:offs[p + 1]]])) if f_sem.shape[1] else 0.0
        tail = np.sum(np.sort(wts)[::-1][k:])
        y, x = divmod(p, w)
        err = np.max(np.abs(full_sem[y, x] - sel_sem[y, x])) if f_sem.shape[1] else 0.0
        if err > max_f * tail + slack:
            return False
    return True


def test_topk_feature_error_bounded_by_tail_mass():
    cam = front_camera(32, 32)
    sc, labels = _stacked_scene()
    full_cfg = RasterConfig(t_min=0.0)
    cache = O.render_cache(sc, labels, cam, full_cfg)
    full = O.render(sc, labels, cam, full_cfg)
    sel = O.render(sc, labels, cam, RasterConfig(t_min=0.0, blending=Blending.TopK, top_k=8))
    assert _tail_bound_holds(cache, sel["sem_feat"], full["sem_feat"], sc.f_sem, 8, 1e-12)
    assert sel["counters"]["blended_total"] < full["counters"]["blended_total"]


# ------------------------------------------------------------ test_raster.cpp:372-390
def _oracle_bench(sc, labels, cam, cfg, binning_precise=Binning.Aabb):
    rows = []
    for name, b, bl in (("baseline", Binning.Circle, Blending.Full), ("precise_tile", binning_precise, Blending.Full),
                        ("topk", Binning.Circle, Blending.TopK), ("full_method", binning_precise, Blending.TopK)):
        c = RasterConfig(**{**cfg.__dict__, "binning": b, "blending": bl})
        best, out = math.inf, None
        for _ in range(2):
            t0 = time.perf_counter()
            out = O.render(sc, labels, cam, c, planes=False)
            best = min(best, time.perf_counter() - t0)
        rows.append({"name": name, "time": best, **out["counters"]})
    return rows


def test_bench_grid_deterministic_counters():
    sc, labels, cam = _street(250, 64, 48, 4)
    r1 = _oracle_bench(sc, labels, cam, RasterConfig())
    r2 = _oracle_bench(sc, labels, cam, RasterConfig())
    for a, b in zip(r1, r2):
        assert a["rn_total"] == b["rn_total"]
        assert a["blended_total"] == b["blended_total"]
    assert r1[1]["rn_total"] <= r1[0]["rn_total"]
    assert r1[2]["blended_total"] == r1[3]["blended_total"]


# ------------------------------------------------------------ acceptance.cpp:33-84 (criterion 1)
@pytest.fixture(scope="module")
def standard_street():
    return _street(12000, 256, 192, 32, seed=7, min_aspect=5.0)


def test_acceptance_1_tile_reduction(standard_street):
    t0 = time.perf_counter()
    sc, labels, cam = standard_street
    cfg = RasterConfig()
    circle = O.bin_surfels(sc.surfels, cam, cfg, 0)
    aabb = O.bin_surfels(sc.surfels, cam, cfg, 1)
    reduction = 1.0 - aabb["rn_total"] / circle["rn_total"]
    a = O.render(sc, labels, cam, RasterConfig(binning=Binning.Circle), planes=False)
    b = O.render(sc, labels, cam, RasterConfig(binning=Binning.Aabb), planes=False)
    max_diff = np.max(np.abs(a["color"] - b["color"]))
    elapsed = time.perf_counter() - t0
    assert reduction >= 0.20 and max_diff < 1e-6 and elapsed < 30.0 and len(sc) >= 1000


# ------------------------------------------------------------ acceptance.cpp:92-167 (criteria 2, 3)
@pytest.mark.slow
def test_acceptance_2_3_topk(standard_street):
    sc, labels, cam = standard_street
    cfg = RasterConfig(top_k=16)
    full_cfg = RasterConfig(top_k=16, binning=Binning.Circle, blending=Blending.Full)
    cache = O.render_cache(sc, labels, cam, full_cfg)
    topk_cfg = RasterConfig(top_k=16, binning=Binning.Circle, blending=Blending.TopK)
    fr = O.render(sc, labels, cam, full_cfg)
    tr = O.render(sc, labels, cam, topk_cfg)
    assert _tail_bound_holds(cache, tr["sem_feat"], fr["sem_feat"], sc.f_sem, 16, 1e-9)
    argmax_frac = np.mean(tr["ins_argmax"] != fr["ins_argmax"])
    assert argmax_frac < 0.02
    rows = _oracle_bench(sc, labels, cam, cfg)
    # criterion 3 counter half: the combined path blends exactly what Top-K blends
    assert rows[3]["blended_total"] == rows[2]["blended_total"]
    # criterion 2's latency half (>= 1.3x) is a wall-clock property of the reference's CPU build on its
    # own machine; on the oracle it is host- and load-dependent, so the deterministic mechanism behind it
    # is asserted instead: Top-K blends strictly fewer feature rows than full blending.
    assert rows[2]["blended_total"] < rows[0]["blended_total"]


# ------------------------------------------------------------ oracle pins of its own
def _ulp_diff(a, b):
    ia = np.asarray(a, dtype=np.float64).view(np.int64)
    ib = np.asarray(b, dtype=np.float64).view(np.int64)
    return np.abs(ia - ib)


def _exp_args():
    rng = np.random.default_rng(0)
    return np.concatenate([
        rng.uniform(-745.2, 709.8, 1_000_000), rng.uniform(-20.0, 0.0, 1_000_000),
        -0.5 * rng.uniform(0, 4.5, 1_000_000) ** 2,            # the alpha range
        rng.uniform(-1100, -500, 100_000), rng.uniform(500, 1100, 100_000),  # special cases
        -np.abs(rng.standard_normal(100_000)) * 1e-15,         # tiny
        [0.0, -0.0, -1e-300, 1e-300, -745.0, -745.2, 709.0, 709.9, -708.5, -700.0, -740.0, -1024.0, 1024.0,
         -512.0, 512.0, np.inf, -np.inf, np.nan, 5e-324, -5e-324]])


def test_psm_exp_is_glibc_exp():
    """psm_exp (paper_2604_10982_b200/csrc/psm_exp.h) restates glibc's exp (called at raster.cpp:390):
    bit-identical to the host glibc on hosts where glibc runs its FMA build (this image and the GPU
    boxes); within 1 ulp elsewhere."""
    xs = _exp_args()
    got, ref = O.psm_exp(xs), O.libm_exp(xs)
    same = (got.view(np.int64) == ref.view(np.int64)) | (np.isnan(got) & np.isnan(ref))
    if O.host_uses_fma_exp():
        assert same.all(), xs[~same][:10]
    else:
        assert np.max(_ulp_diff(got[~np.isnan(ref)], ref[~np.isnan(ref)])) <= 1


def test_psm_exp_through_alpha_closed_form():
    """The alpha path uses it: alpha at (u, v) = (1, 1) is o e^-1 with glibc's exp."""
    cam = front_camera()
    s = facing_surfel((0, 0, 2), 0.1, 0.1, 0.8, (1, 0, 0))
    r = O.evaluate_alpha(s, cam, cam.cx + 5.0, cam.cy + 5.0, RasterConfig())
    x = -0.5 * (r["u"] * r["u"] + r["v"] * r["v"])
    assert _ulp_diff(r["alpha"], 0.8 * math.exp(x)) <= 1


def test_oracle_psm_exp_vs_libm_decisions(standard_street):
    """The oracle built on glibc's exp (what raster.cpp:390 calls) and the one built on psm_exp render the
    standard street scene identically (bit-identical on FMA hosts)."""
    sc, labels, cam = standard_street
    cfg = RasterConfig(blending=Blending.TopK, top_k=16)
    a = O.render(sc, labels, cam, cfg, planes=False)
    b = O.render(sc, labels, cam, cfg, planes=False, libm=True)
    assert np.array_equal(a["blend_count"], b["blend_count"])
    assert a["counters"]["blended_total"] == b["counters"]["blended_total"]
    assert np.max(np.abs(a["color"] - b["color"])) < 1e-12


# ------------------------------------------------------------ Ellipse binning (north-star extension)
def _support_pass_any(finv, center, tile, tiles_x, w, h, ts=16, chi2=9.0):
    tx, ty = tile % tiles_x, tile // tiles_x
    xs = np.arange(tx * ts, min(w, tx * ts + ts)) + 0.5
    ys = np.arange(ty * ts, min(h, ty * ts + ts)) + 0.5
    px, py = np.meshgrid(xs, ys)
    dx = px - center[0]
    dy = py - center[1]
    f00, f01x2, f11 = finv[0, 0], 2.0 * finv[0, 1], finv[1, 1]
    q = f00 * dx * dx + f01x2 * dx * dy + f11 * dy * dy  # raster.cpp:379 operation order
    return bool(np.any(~(q > chi2)))


@pytest.mark.parametrize("which", ["street", "random"])
def test_ellipse_binning_conservative(which):
    """Every (surfel, tile) the Ellipse test drops from the AABB lists has no pixel centre passing the
    support test, so the per-pixel contributor sequences (and every output) are unchanged."""
    if which == "street":
        sc, _, cam = _street(3000, 128, 96, 0)
        rows = sc.surfels
    else:
        cam = front_camera(128, 96)
        rows = np.array(_random_surfels(21, 300, 0.01, 0.8))
    cfg = RasterConfig()
    aabb = O.bin_surfels(rows, cam, cfg, 1)
    ell = O.bin_surfels(rows, cam, cfg, 2)
    tiles_x = (cam.width + 15) // 16
    assert ell["rn_total"] < aabb["rn_total"]
    proj = {}
    for t, (la, le) in enumerate(zip(aabb["tiles"], ell["tiles"])):
        sa, se = set(la.tolist()), set(le.tolist())
        assert se <= sa
        for s in sa - se:
            if s not in proj:
                proj[s] = O.project_surfel(rows[s], cam)
            p = proj[s]
            assert not _support_pass_any(p["footprint_inv"], p["center"], t, tiles_x, cam.width, cam.height), (s, t)


def test_ellipse_render_identical_to_aabb(standard_street):
    sc, labels, cam = standard_street
    for blending in (Blending.Full, Blending.TopK):
        a = O.render(sc, labels, cam, RasterConfig(binning=Binning.Aabb, blending=blending))
        e = O.render(sc, labels, cam, RasterConfig(binning=Binning.Ellipse, blending=blending))
        for k in ("color", "depth", "normal", "sem_feat", "ins_dist", "ins_argmax", "alpha_acc", "blend_count"):
            assert np.array_equal(a[k], e[k]), k
        assert a["counters"]["blended_total"] == e["counters"]["blended_total"]
        assert e["counters"]["rn_total"] < a["counters"]["rn_total"]


def test_topk_select_semantics():
    """topk_select (raster.cpp:225-251): k >= m selects all; ties go to the lower proj index."""
    w = [0.1, 0.3, 0.3, 0.2, 0.3]
    sel = O.topk_select(w, [0, 1, 2, 3, 4], 2)
    assert sel.tolist() == [False, True, True, False, False]
    assert O.topk_select(w, [0, 1, 2, 3, 4], 5).all()
    assert O.topk_select(w, [0, 1, 2, 3, 4], 9).all()
