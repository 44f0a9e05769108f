"""GPU: asynchronous frame chains and the pipelined view batch (psm_render_batch, the C5 view-batch
config of SURVEY.md §8d/e) give the same planes as one synchronous render per view, including when
frames outgrow the context's buffers and psm_sync re-renders them."""
import numpy as np
import pytest

from paper_2604_10982_b200 import (Binning, Blending, Camera, RasterConfig, Renderer, StreetSpec, density_scale,
                                   make_street_scene, trajectory_cameras)

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

W, H, C_SEM = 256, 192, 16
NAMES = ("color", "depth", "normal", "sem_feat", "ins_argmax", "alpha_acc", "blend_count")
CH = {"color": 3, "depth": 2, "normal": 3, "sem_feat": C_SEM, "ins_argmax": 1, "alpha_acc": 1, "blend_count": 1}


@pytest.fixture(scope="module")
def street():
    n = 12000
    sc, _, cam0 = make_street_scene(StreetSpec(n_surfels=n, image_w=W, image_h=H, c_sem=C_SEM,
                                               scale_mult=density_scale(n, W, H)), with_labels=False)
    return sc, [cam0] + trajectory_cameras(256, W, H, first=40, count=6)


def away_camera():
    """Looks away from the street (every surfel culled): the first frame sizes the key buffers
    to almost nothing, so the frames after it overflow them."""
    return Camera.look_at((0.0, 0.0, 0.0), (0.0, 0.0, -20.0), (0.0, -1.0, 0.0), 0.8 * W, 0.8 * W, W, H, 0.1, 200.0)


def device_planes():
    dev = torch.device("cuda", 0)
    out = {}
    for k in NAMES:
        dt = torch.int32 if k in ("ins_argmax", "blend_count") else torch.float32
        out[k] = torch.full((H * W * CH[k],), -7, dtype=dt, device=dev)
    return out


def ptrs(p):
    return {k: v.data_ptr() for k, v in p.items()}


def assert_same(planes, ref):
    for k in NAMES:
        got = planes[k].cpu().numpy().reshape(H, W, CH[k])
        assert np.array_equal(got, getattr(ref, k)), k


CFG = RasterConfig(binning=Binning.Ellipse, blending=Blending.TopK, top_k=8)


def references(street):
    sc, cams = street
    r = Renderer(0)
    try:
        return [r.render(sc, None, c, CFG) for c in cams]
    finally:
        r.close()


def test_gpu_async_chain_rerenders_overflowed_frames(street):
    sc, cams = street
    refs = references(street)
    r = Renderer(0)
    try:
        ds = r.upload(sc)
        cnt = r.render_device(ds, away_camera(), CFG, ptrs(device_planes()), counters=True)
        assert cnt.rn_total == 0
        planes = [device_planes() for _ in cams]
        for c, p in zip(cams, planes):  # asynchronous: every one outgrows the key buffers sized above
            r.render_device(ds, c, CFG, ptrs(p))
        last = r.sync()
        for p, ref in zip(planes, refs):
            assert_same(p, ref)
        assert last.rn_total == refs[-1].rn_total and last.blended_total == refs[-1].blended_total
    finally:
        r.close()


def test_gpu_async_chain_shared_planes_end_as_the_last_frame(street):
    sc, cams = street
    refs = references(street)
    r = Renderer(0)
    try:
        ds = r.upload(sc)
        r.render_device(ds, away_camera(), CFG, ptrs(device_planes()), counters=True)
        shared = device_planes()
        for c in cams:  # the re-render of an early overflowed frame must not survive the later ones
            r.render_device(ds, c, CFG, ptrs(shared))
        r.sync()
        assert_same(shared, refs[-1])
    finally:
        r.close()


@pytest.mark.parametrize("fresh", [True, False])
def test_gpu_render_batch_matches_single_views(street, fresh):
    """Odd view count (the context renders views 0, 2, .., its twin 1, 3, ..); `fresh` makes both
    contexts start with undersized buffers (every view overflows and is re-rendered at psm_sync)."""
    sc, cams = street
    refs = references(street)
    r = Renderer(0)
    try:
        ds = r.upload(sc)
        if fresh:
            r.render_device(ds, away_camera(), CFG, ptrs(device_planes()), counters=True)
        else:
            for c in cams:
                r.render_device(ds, c, CFG, ptrs(device_planes()), counters=True)
        for rep in range(2):
            planes = [device_planes() for _ in cams]
            r.render_batch_device(ds, cams, CFG, [ptrs(p) for p in planes])
            last = r.sync()
            for p, ref in zip(planes, refs):
                assert_same(p, ref)
            assert last.rn_total == refs[-1].rn_total and last.n_proj == refs[-1].n_proj
        # work queued on the context stream after a batch sees every view (the batch joins it)
        planes = [device_planes() for _ in cams[:4]]
        r.render_batch_device(ds, cams[:4], CFG, [ptrs(p) for p in planes])
        after = r.render(sc, None, cams[0], CFG)  # synchronous: drains the batch first
        for p, ref in zip(planes, refs[:4]):
            assert_same(p, ref)
        for k in NAMES:
            assert np.array_equal(getattr(after, k), getattr(refs[0], k)), k
    finally:
        r.close()
