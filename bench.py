"""Benchmark of the Ψ-Map render hot path on B200 (BASELINE.json metric: panoptic frames/s at
1M surfels, 1280x720, 64-d features, K=8; % HBM roofline).

One step = one full render of one view (K1 preprocess .. K7 blend) of the C3 workload: the
density-normalised street scene with 1M surfels, 1280x720, C_sem = 64, Top-K = 8,
Ellipse (precise) binning, synthetic data. Multi-GPU: one process per GPU, each renders its own
views of a replicated scene (weak scaling, no collective on the render path).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c3|c2|c4|c1]
"""
import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (n_surfels, W, H, c_sem, blending, K, description)
    "c1": (10_000, 256, 256, 0, "full", 16, "10k surfels 256x256 RGB+depth"),
    "c2": (1_000_000, 1280, 720, 0, "full", 16, "1M surfels 1280x720 RGB+depth+normal"),
    "c3": (1_000_000, 1280, 720, 64, "topk", 8, "1M surfels 1280x720 64-d semantics Top-K=8"),
    "c3p": (1_000_000, 1280, 720, 64, "topk", 8, "render_panoptic over 1M surfels 1280x720 64-d semantics, "
                                                 "32 instance queries (assign_labels each frame), Top-K=8"),
    "c4": (5_000_000, 1920, 1080, 128, "topk", 16, "5M surfels 1920x1080 128-d semantics Top-K=16"),
    "c5": (5_000_000, 1920, 1080, 128, "topk", 16, "256-view trajectory over 5M surfels 1920x1080 128-d Top-K=16, "
                                                     "views sharded across ranks"),
}
C5_VIEWS = 256
METRIC = "panoptic frames/s at 1M surfels, 1280x720, 64-d feats, K=8; % HBM roofline"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def alg_bytes(n, n_proj, w, h, c):
    """B_alg = 52 N + 4 C N_proj + W H (44 + 4 C) (fp32-equivalent compulsory traffic)."""
    frame = 52 * n + 4 * c * n_proj + w * h * (44 + 4 * c)
    blend = 4 * c * n_proj + w * h * (44 + 4 * c)  # the blend kernel's share (features read, planes written)
    return frame, blend


class ClockSampler:
    """SM clocks and throttle reasons polled through NVML every 2 ms during the timed region (the
    B200_PROFILING.md clocks line; nvidia-smi's 100 ms period is longer than a short timed region)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, device):
        self.device = device
        self.samples = []
        self.stop = threading.Event()
        self.handle = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        except Exception as e:  # no NVML: report unsampled
            log(f"clock sampler unavailable: {e}")
            self.handle = None
        return self

    def _poll(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
                self.samples.append((mhz, rs))
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *exc):
        self.stop.set()
        if self.handle is not None:
            self.t.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted({name for _, rs in self.samples for name, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": statistics.median(m for m, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples)}


C3P_QUERIES = 32


def build_workload(name, rank, world):
    from paper_2604_10982_b200 import (SceneMap, StreetSpec, density_scale, make_street_scene, street_f_ins,
                                       street_queries, trajectory_cameras)
    n, w, h, c, blending, k, desc = WORKLOADS[name]
    t0 = time.perf_counter()
    spec = StreetSpec(n_surfels=n, image_w=w, image_h=h, c_sem=c, scale_mult=density_scale(n, w, h))
    scene, _, cam0 = make_street_scene(spec, with_labels=False)
    if name == "c3p":  # the panoptic layer's inputs: Surfel::f_ins and synthetic instance queries
        scene = SceneMap(scene.surfels, scene.f_sem, street_f_ins(spec), street_queries(C3P_QUERIES))
    cams, _ = rank_cameras(name, cam0, rank, world)
    log(f"[rank {rank}] workload {name}: {len(scene)} surfels generated in {time.perf_counter() - t0:.1f}s")
    return scene, cams, (n, w, h, c, blending, k, desc)


def rank_cameras(name, cam0, rank, world):
    """The views rank `rank` of `world` renders each step, and their trajectory indices.
    c5: the rank's contiguous block of the closed-form 256-view trajectory.
    Other workloads (weak scaling): rank r renders trajectory view r (view 0 is the street camera)."""
    from paper_2604_10982_b200 import trajectory_cameras
    from paper_2604_10982_b200.multiview import shard_range
    _, w, h = WORKLOADS[name][:3]
    if name == "c5":
        views = list(shard_range(C5_VIEWS, world, rank))
        return (trajectory_cameras(C5_VIEWS, w, h, first=views[0], count=len(views)) if views else []), views
    return [cam0 if rank == 0 else trajectory_cameras(1, w, h, first=rank, count=1)[0]], [rank]


def raster_cfg(blending, k, reference=False):
    """GPU arm: Ellipse (exact precise-tile) binning. Reference arm: the reference's own precise binning,
    bin_aabb (raster.cpp:149-152), i.e. its `full_method` row (raster.cpp:525). Outputs are identical."""
    from paper_2604_10982_b200 import Binning, Blending, RasterConfig
    return RasterConfig(binning=Binning.Aabb if reference else Binning.Ellipse,
                        blending=Blending.TopK if blending == "topk" else Blending.Full, top_k=k)


def reference_workload(name):
    """The reference arm's inputs, built without the product library: the oracle's restatement of
    make_street_scene (+ scale_mult), pinned bit-exact to the reference's own generator by
    tests/test_ref_pin.py. Returns (surfels13, f_sem, psm_camera, (n, w, h, c, blending, k, desc))."""
    from oracle import pyoracle as O
    from paper_2604_10982_b200.scene import StreetSpec, density_scale  # plain dataclass + formula
    n, w, h, c, blending, k, desc = WORKLOADS[name]
    t0 = time.perf_counter()
    spec = StreetSpec(n_surfels=n, image_w=w, image_h=h, c_sem=c, scale_mult=density_scale(n, w, h))
    if name == "c3p":
        s, f, _, cam, fi = O.make_street_scene(spec, with_f_ins=True)
    else:
        s, f, _, cam = O.make_street_scene(spec)
        fi = None
    log(f"[reference] workload {name}: {s.shape[0]} surfels generated by the oracle in {time.perf_counter() - t0:.1f}s")
    return s, f, fi, cam, (n, w, h, c, blending, k, desc)


def repo_libs():
    """The repo's shared libraries mapped into this process (evidence of what a timed arm ran)."""
    try:
        return sorted({ln.split()[-1].replace(ROOT + "/", "") for ln in open("/proc/self/maps")
                       if ln.rstrip().endswith(".so") and ROOT in ln})
    except OSError:
        return []


class CpuReference:
    """The reference CPU renderer on the host cores. Preferred: oracle/_ref, the reference's own
    sources compiled unchanged (kind "reference"): render_into into persistent targets (raster.cpp /
    math_util.cpp / core_types.cpp: serial project + bin, std::thread tile loop, raster.cpp:273-511,
    glibc exp), or for c3p render_panoptic (metrics.cpp:339-369 with panoptic.cpp's assign_labels)
    over a scene built once. Where _ref is absent: the oracle restatement built with glibc exp
    (kind "port")."""

    def __init__(self, surfels, f_sem, f_ins=None, queries=None):
        from oracle import pyref as R
        from paper_2604_10982_b200.raster import SceneMap
        self.queries = queries
        self.kind = "reference" if R.available() else "port"
        if self.kind == "reference":
            self.rs = (R.RefPanopticScene(SceneMap(surfels, f_sem, f_ins, queries)) if queries
                       else R.RefScene(surfels, f_sem, None))
        else:
            self.scene = SceneMap(surfels, f_sem, f_ins, queries)

    def frame(self, cam_c, cfg):
        if self.kind == "reference":
            if self.queries:
                self.rs.render(cam_c, cfg.to_c())
            else:
                self.rs.render_into(cam_c, cfg.to_c())
            return
        from oracle import pyoracle as O
        from paper_2604_10982_b200.raster import Camera
        cam = Camera.from_c(cam_c)
        if self.queries:  # render_panoptic (metrics.cpp:339-369): assign_labels + render + epilogue
            O.render_panoptic(self.scene, self.scene.f_ins, self.queries, cam, cfg)
        else:
            O.render(self.scene, None, cam, cfg, planes=False, libm=True)

    def time(self, cam_c, cfg, frames):
        times = []
        for _ in range(frames):
            t0 = time.perf_counter()
            self.frame(cam_c, cfg)
            times.append(time.perf_counter() - t0)
        return times

    def describe(self, frames, w, h, n, threads):
        if self.kind == "reference" and self.queries:
            what = ("the reference's render_panoptic (metrics.cpp with panoptic.cpp's assign_labels and raster.cpp's "
                    "render) compiled unchanged (oracle/_ref, minimal Eigen stand-in), scene built once")
        elif self.kind == "reference":
            what = ("the reference's raster.cpp/math_util.cpp/core_types.cpp compiled unchanged (oracle/_ref, "
                    "minimal Eigen stand-in), render_into into persistent targets")
        else:
            what = "reference algorithm restated in C++ (oracle), glibc exp"
        return (f"{frames} full {w}x{h} frames of {n} surfels, best-of; {what}; serial project+bin, "
                f"{threads} std::threads over tiles")


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return 0
    s, f, fi, cam_c, (n, w, h, c, blending, k, desc) = reference_workload(args.workload)
    queries = None
    if args.workload == "c3p":
        from paper_2604_10982_b200.panoptic import street_queries
        queries = street_queries(C3P_QUERIES)
    ref = CpuReference(s, f, fi, queries)
    cfg = raster_cfg(blending, k, reference=True)
    ref.time(cam_c, cfg, args.warmup)
    times = ref.time(cam_c, cfg, args.steps)
    fps = 1.0 / min(times)
    threads = int(os.environ.get("PSIMAP_THREADS", 0)) or os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * statistics.mean(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.workload}: {desc}", "binning": "aabb (reference full_method)",
                   "cpu_only": True, "same_config_note": "AABB here vs Ellipse on the GPU: identical planes "
                   "(tests/test_gpu_parity.py::test_gpu_c3_binning_output_identity)"},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": threads, "kind": ref.kind,
                         "sample": ref.describe(args.steps, w, h, n, threads)},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "libs_loaded": repo_libs(),
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import numpy as np
    import torch

    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    from paper_2604_10982_b200 import Renderer
    from paper_2604_10982_b200 import _abi as A

    scene, cams, (n, w, h, c, blending, k, desc) = build_workload(args.workload, rank, world)
    cam = cams[0]
    cfg = raster_cfg(blending, k)
    stream = torch.cuda.Stream(device=dev)
    r = Renderer(local_rank, stream=stream.cuda_stream)
    pano = bool(scene.queries)  # c3p: render_panoptic (assign_labels + fused panoptic blend) per frame
    t0 = time.perf_counter()
    ds = r.upload(scene, exact=pano)
    qclass = np.array([q.class_id for q in scene.queries], np.int32)
    if pano:
        r.assign_labels(ds, scene.queries)
    torch.cuda.synchronize()
    upload_s = time.perf_counter() - t0
    npx = w * h
    planes_t = {
        "color": torch.empty(npx * 3, dtype=torch.float32, device=dev),
        "depth": torch.empty(npx * 2, dtype=torch.float32, device=dev),
        "normal": torch.empty(npx * 3, dtype=torch.float32, device=dev),
        "sem_feat": torch.empty(max(npx * c, 1), dtype=torch.float32, device=dev),
        "ins_argmax": torch.empty(npx, dtype=torch.int32, device=dev),
        "alpha_acc": torch.empty(npx, dtype=torch.float32, device=dev),
        "blend_count": torch.empty(npx, dtype=torch.int32, device=dev),
    }
    if pano:
        planes_t = {kk: torch.empty(npx, dtype=torch.int32, device=dev) for kk in ("ids", "classes", "sem_classes")}
    ptrs = {kk: v.data_ptr() for kk, v in planes_t.items()}
    batch = len(cams) > 1  # c5: the rank's views as one pipelined psm_render_batch per step
    if batch:  # views alternate between two contexts; each context reuses one plane set
        ptrs2 = {kk: torch.empty_like(v).data_ptr() for kk, v in planes_t.items()}
        batch_ptrs = [ptrs if i % 2 == 0 else ptrs2 for i in range(len(cams))]

    def frame(cv, counters):
        if pano:  # psimap::render_panoptic: assign_labels, then the render with the fused epilogue
            r.assign_labels(ds, scene.queries, outputs=False)
            return r.render_panoptic_device(ds, cv, cfg, qclass, ptrs, counters=counters)
        return r.render_device(ds, cv, cfg, ptrs, counters=counters)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    # warm-up (also sizes every grow-only buffer)
    r.set_profiling(True)
    cnt = None
    for _ in range(max(args.warmup, 1)):
        if batch:  # every view once: both contexts' buffers sized for the whole trajectory
            r.render_batch_device(ds, cams, cfg, batch_ptrs)
            cnt = r.sync()
        else:
            cnt = frame(cam, True)
    n_proj = int(cnt.n_proj)

    # timed region: per step, flush L2 (outside the events), then one render between events on its stream
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    blend_ms, stage = [], []
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
                ev[i][0].record(stream)
            if batch:
                r.render_batch_device(ds, cams, cfg, batch_ptrs)
            else:
                frame(cam, False)
            with torch.cuda.stream(stream):
                ev[i][1].record(stream)
            r.sync()
            st = r.stage_times()  # batch: the stages of the last view (the views overlap in pairs)
            blend_ms.append(st["blend"])
            stage.append(st)
        torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    r.set_profiling(False)
    cnt = r.sync()
    assign_ms = None
    if pano:  # assign_labels alone, device-timed on the render stream
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
        for _ in range(5):
            r.assign_labels(ds, scene.queries, outputs=False)
        with torch.cuda.stream(stream):
            e1.record(stream)
        torch.cuda.synchronize()
        assign_ms = e0.elapsed_time(e1) / 5

    # e2e through the C-ABI with host (pinned) targets: D2H of every plane inside each step. Every
    # rank renders its own view at once (each GPU its own PCIe link); the value is the frames of all
    # ranks over the slowest rank's wall time per step.
    e2e = None

    def e2e_barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def e2e_max(sec):
        if world > 1:
            t_ = torch.tensor([sec], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(t_, op=torch.distributed.ReduceOp.MAX)
            sec = float(t_.item())
        return sec
    if pano:
        from paper_2604_10982_b200.panoptic import PanopticRender
        pr = PanopticRender(*(torch.empty((h, w, 1), dtype=torch.int32, pin_memory=True).numpy() for _ in range(3)))
        r.render_panoptic(ds, cam, cfg, qclass, out=pr)  # warm
        torch.cuda.synchronize()
        e2e_steps = max(3, min(args.steps, 10))
        e2e_barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            r.assign_labels(ds, scene.queries, outputs=False)
            r.render_panoptic(ds, cam, cfg, qclass, out=pr)
        e2e_s = e2e_max((time.perf_counter() - t0) / e2e_steps)
        e2e = {"value": world / e2e_s, "unit": "frames/s", "h2d_bytes_per_step": C.sizeof(A.psm_camera),
               "d2h_bytes_per_step": int(pr.ids.nbytes + pr.classes.nbytes + pr.sem_classes.nbytes),
               "steps": e2e_steps,
               "note": "assign_labels (async) + psm_render_panoptic with host targets: the three int32 id planes "
                       "copied back per frame to pinned memory; scene resident (exact fp64 features, upload "
                       f"{upload_s * 1000:.0f} ms once)"}
    elif rank == 0 or world > 1:
        from paper_2604_10982_b200.raster import RenderTargets
        host = RenderTargets()
        host.ensure(w, h, c, 0)
        pinned = {}
        for name in ("color", "depth", "normal", "sem_feat", "ins_argmax", "alpha_acc", "blend_count"):
            a = getattr(host, name)
            t_ = torch.empty(a.shape, dtype=torch.float32 if a.dtype == np.float32 else torch.int32,
                             pin_memory=True)
            pinned[name] = t_
            setattr(host, name, t_.numpy())
        host.ins_dist = np.zeros((h, w, 0), np.float32)
        r.render_into(host, ds, None, cam, cfg)  # warm
        torch.cuda.synchronize()
        e2e_steps = max(3, min(args.steps, 10))
        e2e_barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            r.render_into(host, ds, None, cam, cfg)
        e2e_s = e2e_max((time.perf_counter() - t0) / e2e_steps)
        d2h = sum(getattr(host, nm).nbytes for nm in ("color", "depth", "normal", "sem_feat", "ins_argmax",
                                                      "alpha_acc", "blend_count"))
        e2e = {"value": world / e2e_s, "unit": "frames/s", "h2d_bytes_per_step": C.sizeof(A.psm_camera),
               "d2h_bytes_per_step": int(d2h), "steps": e2e_steps,
               "note": "psm_render with host targets: camera to device (kernel arguments), full render, "
                       "cudaMemcpy of all planes to pinned host memory; every rank at once, all ranks' frames "
                       "over the slowest rank's wall time; scene resident (upload "
                       f"{upload_s * 1000:.0f} ms once)"}

    if rank != 0:
        if world > 1:
            torch.distributed.barrier()
            torch.distributed.destroy_process_group()
        return 0

    views_total = C5_VIEWS if args.workload == "c5" else world
    frames = args.steps * views_total
    value = frames / (total_ms / 1000.0)
    b_frame, b_blend = alg_bytes(n, n_proj, w, h, c)
    if pano:  # fp64 feature + label rows read; 44 B/px of planes plus 12 B/px of ids written
        d = c + len(scene.queries)
        b_blend = 8 * d * n_proj + w * h * 56
        b_frame = 52 * n + 64 * n + 12 * len(scene.queries) * n + b_blend
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = peaks.get("hbm_gbs", 6650.0)
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    blend_avg = statistics.mean(blend_ms)
    achieved = b_blend / (blend_avg / 1000.0) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "blend_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    stage_avg = {kk: statistics.mean(s[kk] for s in stage) for kk in stage[0]}

    # CPU baseline on rank 0 at N=1: the reference algorithm on the host cores, bounded sample
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        ref = CpuReference(scene.surfels, scene.f_sem, scene.f_ins, scene.queries or None)
        times = ref.time(cam.to_c(), raster_cfg(blending, k, reference=True), 2)
        threads = int(os.environ.get("PSIMAP_THREADS", 0)) or os.cpu_count()
        cpu = {"value": 1.0 / min(times), "unit": "frames/s", "cores": threads, "kind": ref.kind,
               "sample": ref.describe(2, w, h, n, threads)}

    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64-decisions/f32-accum", "data": "synthetic",
        "dtype_note": "projection, culling, binning, sort keys, support/alpha/transmittance and Top-K decisions in "
                      "fp64 (bit-exact with the reference); colour/normal/feature sums in fp32 (1e-4 tolerance)",
        "config": {"workload": f"{args.workload}: {desc}", "binning": "ellipse (precise tile intersection)",
                   "queries": len(scene.queries), "assign_labels_ms": assign_ms,
                   "blending": blending, "top_k": k, "surfels": n, "n_proj": n_proj, "width": w, "height": h,
                   "c_sem": c, "rn_total": int(cnt.rn_total), "blended_total": int(cnt.blended_total),
                   "l2": "flushed between timed steps (256 MB write outside the events)",
                   "views_per_rank_per_step": len(cams),
                   "parallelism": f"view-sharded x{world}, scene replicated",
                   "stage_ms": stage_avg, "alg_bytes_per_frame": b_frame,
                   **({"stage_ms_note": "batch: event spans of the last view of each step; its stages share the "
                                        "GPU with the other context's view, so front-end spans include waits "
                                        "(tile_scan most)"} if batch else {})},
        "roofline": {"bound": "hbm", "kernel": "blend_kernel (K7)", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "peak_source": peak_src, "alg_bytes_per_launch": b_blend, "launch_ms": blend_avg},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": (12 if pano else 11) * args.steps * len(cams),
        "gpu_launches_note": "per frame: frame_init, preprocess, tile_sub_scan, tile_scan, emit, sort_tiles_huge, "
                             "sort_tiles<1024,3>, sort_tiles<1024,2>, sort_tiles<512,1>, sort_tiles<128,0>, blend "
                             "(+1 small D2H of the counters)" + ("; c3p adds assign_labels" if pano else "")
                             + ("; c5: one psm_render_batch per step, views alternating over two streams"
                                if batch else ""),
        "clocks": clk.summary(),
        "libs_loaded": repo_libs(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return 0


def run_grid(args):
    """The reference's bench_render ablation grid (raster.cpp:513-573, Table 3 rows) on the GPU, plus
    the Ellipse (exact precise-tile) rows: one JSON line with every row (min of `steps` device times)."""
    import torch
    from paper_2604_10982_b200 import Binning, Renderer, bench_render
    torch.cuda.set_device(0)
    scene, cams, (n, w, h, c, blending, k, desc) = build_workload(args.workload, 0, 1)
    r = Renderer(0, stream=torch.cuda.current_stream().cuda_stream)
    ds = r.upload(scene)
    out = {"grid": args.workload, "desc": desc, "top_k": k, "rows": []}
    for precise in (Binning.Aabb, Binning.Ellipse):
        rep = bench_render(ds, None, cams[0], max(args.steps, 1), raster_cfg(blending, k), renderer=r,
                           binnings=precise)
        for row in rep.rows:
            if precise == Binning.Ellipse and row.binning == Binning.Circle:
                continue
            out["rows"].append({"name": row.name if precise == Binning.Aabb else row.name + "_ellipse",
                                "binning": row.binning.name, "blending": row.blending.name,
                                "time_ms": row.time_ms, "fps": row.fps, "rn_total": row.rn_total,
                                "rn_per_tile": row.rn_per_tile, "blended_total": row.blended_total,
                                "blended_per_pixel": row.blended_per_pixel})
    print(json.dumps(out), flush=True)
    return 0


def spawn_ranks(args):
    """`--gpus N` without a torchrun environment: re-launch this command as N ranks (one process
    per GPU) under torch.distributed.run, exactly as the driver's multi-GPU launch does."""
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    log(f"spawning {args.gpus} ranks: {' '.join(cmd)}")
    return subprocess.call(cmd)


def run_dry(args):
    """--dry-run: the multi-rank plumbing of run_ours on CPU (gloo), without a device: process group,
    per-rank views, barrier, per-rank step timing, MAX over ranks, one JSON line from rank 0. Frames are
    not rendered (no GPU); used by tests/test_bench_ranks.py to exercise `--gpus N` end to end."""
    import torch
    import torch.distributed as dist
    rank, _, world = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    from paper_2604_10982_b200 import Camera
    n, w, h, c, blending, k, desc = WORKLOADS[args.workload]
    cam0 = Camera.look_at((0, 0, 0), (0, 0, 20), (0, -1, 0), 0.8 * w, 0.8 * w, w, h, 0.1, 200.0)
    cams, views = rank_cameras(args.workload, cam0, rank, world)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for cv in cams:
            cv.to_c()  # the per-view kernel arguments; no render without a device
    total_ms = (time.perf_counter() - t0) * 1000.0
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        gathered = [None] * world
        dist.all_gather_object(gathered, {"rank": rank, "views": views,
                                          "t_cw": [[float(x) for x in cv.t_cw] for cv in cams[:1]]})
    else:
        gathered = [{"rank": 0, "views": views}]
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": total_ms / max(args.steps, 1),
                          "config": {"workload": f"{args.workload}: {desc}"}, "ranks": gathered}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--grid", action="store_true", help="print the bench_render ablation grid instead")
    ap.add_argument("--dry-run", action="store_true", help="rank plumbing on CPU (gloo), no device work")
    args = ap.parse_args()
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1 and args.impl == "ours" and not args.grid:
        return spawn_ranks(args)
    if env_world is not None and args.impl == "ours" and int(env_world) != args.gpus:
        log(f"WORLD_SIZE={env_world} does not match --gpus {args.gpus}")
        return 2
    if args.dry_run:
        return run_dry(args)
    if args.grid:
        return run_grid(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
