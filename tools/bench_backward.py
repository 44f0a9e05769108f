"""Times the GPU render backward (psm_render_backward) at a bench workload.

  python tools/bench_backward.py [workload] [reps]

Prints the wall time per call (which includes the host->device copy of the upstream
plane gradients and the device->host copy of every surfel gradient). The kernel times
are read from an ncu launch list of the same command, e.g.
  ncu --metrics gpu__time_duration.sum -k regex:"backward|blend" python tools/bench_backward.py c3 1
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2604_10982_b200 import Renderer  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
scene, cams, (n, w, h, c, blending, k, desc) = bench.build_workload(wl, 0, 1)
cfg = bench.raster_cfg(blending, k)
r = Renderer(0)
rng = np.random.default_rng(1)
gc = rng.normal(size=(h, w, 3))
gs = rng.normal(size=(h, w, c)) if c else None
for i in range(reps):
    t0 = time.perf_counter()
    g = r.render_backward(scene, None, cams[0], cfg, gc, gs, None)
    print(f"{wl} rep {i}: {1000 * (time.perf_counter() - t0):.1f} ms wall; sum|d_color| {np.abs(g['color']).sum():.6e} "
          f"sum|d_center| {np.abs(g['center']).sum():.6e}")
