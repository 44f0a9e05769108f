"""One device-resident frame of a bench workload, for ncu (python profiles/frame.py [c3|c4|...] [frames]).

Renders `frames` frames (default 2; the first sizes the context's buffers); summarize.py
keeps the launches of the last one."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2604_10982_b200 import Renderer  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 2
scene, cams, (n, w, h, c, blending, k, desc) = bench.build_workload(wl, 0, 1)
r = Renderer(0)
pano = bool(scene.queries)  # c3p: assign_labels + render_panoptic, as bench.py's step
ds = r.upload(scene, exact=pano)
cfg = bench.raster_cfg(blending, k)
if pano:
    import numpy as np
    import torch
    qclass = np.array([q.class_id for q in scene.queries], np.int32)
    ptrs = {kk: torch.empty(w * h, dtype=torch.int32, device="cuda:0").data_ptr()
            for kk in ("ids", "classes", "sem_classes")}
for _ in range(frames):
    if pano:
        r.assign_labels(ds, scene.queries, outputs=False)
        r.render_panoptic_device(ds, cams[0], cfg, qclass, ptrs)
    else:
        r.render_device(ds, cams[0], cfg, {})  # NULL planes: context scratch
    r.sync()
print(f"{wl}: {frames} frames rendered")
