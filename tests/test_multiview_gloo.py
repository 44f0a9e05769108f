"""Multi-rank view sharding on CPU (gloo, world_size 2): every view is rendered exactly once,
counters combine to the single-process result, time is the max over ranks. The renderer is the
CPU oracle here (no GPU in this container); bench.py runs the same path with the GPU renderer."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_10982_b200.multiview import combine, gather_results, run_shard, shard_range


def test_shard_range_partitions_views():
    for n in (0, 1, 7, 256):
        for world in (1, 2, 3, 8):
            seen = [v for r in range(world) for v in shard_range(n, world, r)]
            assert seen == list(range(n))
            sizes = [len(shard_range(n, world, r)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _views():
    from paper_2604_10982_b200 import trajectory_cameras
    return trajectory_cameras(6, 64, 48, first=0, count=6, total=6)


def _render_fn():
    from oracle import pyoracle as O
    from paper_2604_10982_b200 import RasterConfig, StreetSpec, make_street_scene
    sc, _, _ = make_street_scene(StreetSpec(n_surfels=600, image_w=64, image_h=48, c_sem=4, n_instances=8),
                                 with_labels=False)
    cfg = RasterConfig()

    def fn(v, cam):
        c = O.render(sc, None, cam, cfg, planes=False)["counters"]
        return {"rn_total": c["rn_total"], "blended_total": c["blended_total"], "n_proj": c["n_proj"]}
    return fn


def _worker(rank, world, port, q):
    import time
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = run_shard(_views(), world, rank, _render_fn(), time.perf_counter)
        allr = gather_results(res)
        if rank == 0:
            q.put(combine(allr))
    finally:
        dist.destroy_process_group()


def test_two_rank_view_sharding_matches_single_process():
    import time
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    single = combine([run_shard(_views(), 1, 0, _render_fn(), time.perf_counter)])
    assert out["views"] == 6
    assert out["counters"] == single["counters"]
    assert out["time_s"] > 0


def test_combine_rejects_duplicates():
    from paper_2604_10982_b200.multiview import ShardResult
    a = ShardResult(0, [0, 1], [{}, {}], 1.0)
    b = ShardResult(1, [1], [{}], 2.0)
    with pytest.raises(ValueError):
        combine([a, b])
    c = ShardResult(1, [2], [{}], 2.0)
    assert combine([a, c])["time_s"] == 2.0
