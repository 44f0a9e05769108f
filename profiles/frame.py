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
ds = r.upload(scene, None)
cfg = bench.raster_cfg(blending, k)
for _ in range(frames):
    r.render_device(ds, cams[0], cfg, {})  # NULL planes: context scratch
    r.sync()
print(f"{wl}: {frames} frames rendered")
