"""View-sharded multi-GPU rendering: one process per GPU, the scene
replicated on every device, the camera views partitioned into contiguous blocks, no
collective on the render path. Views are independent in the reference
(proj/src/raster.cpp:273-511 reads only the scene and one camera), so each rank
renders its block alone; only per-view counters and the timing are combined on the
host after the timed region (all_gather of counters, MAX of elapsed time: the
whole-job time is the slowest rank's).

`render_fn(view_index, camera) -> dict of counters` is injected: the benchmark passes
the GPU renderer, the CPU multi-rank tests pass a stand-in.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Dict, List, Sequence


def shard_range(n_views: int, world: int, rank: int) -> range:
    """Contiguous block of views of `rank` out of `world` (sizes differ by at most one)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n_views, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


@dataclass
class ShardResult:
    rank: int
    views: List[int]
    counters: List[Dict[str, float]]
    elapsed_s: float


def run_shard(cams: Sequence, world: int, rank: int, render_fn: Callable[[int, object], Dict[str, float]],
              clock: Callable[[], float]) -> ShardResult:
    views = list(shard_range(len(cams), world, rank))
    t0 = clock()
    counters = [render_fn(v, cams[v]) for v in views]
    return ShardResult(rank, views, counters, clock() - t0)


def combine(results: Sequence[ShardResult]) -> Dict[str, object]:
    """Whole-job view of the per-rank results: every view exactly once, counters in view
    order, time = max over ranks, frames/s = views / time."""
    by_view = {}
    for r in results:
        for v, c in zip(r.views, r.counters):
            if v in by_view:
                raise ValueError(f"view {v} rendered twice")
            by_view[v] = c
    n = len(by_view)
    if sorted(by_view) != list(range(n)):
        raise ValueError("views missing")
    t = max(r.elapsed_s for r in results)
    return {"views": n, "time_s": t, "frames_per_s": n / t if t > 0 else float("inf"),
            "counters": [by_view[v] for v in range(n)]}


def gather_results(local: ShardResult) -> List[ShardResult]:
    """Host-side all_gather of the per-rank results (torch.distributed, any backend)."""
    import torch.distributed as dist
    world = dist.get_world_size()
    out: List[object] = [None] * world
    dist.all_gather_object(out, local)
    return out  # type: ignore[return-value]
