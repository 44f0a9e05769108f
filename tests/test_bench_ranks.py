"""bench.py's launcher and arms on CPU: `--gpus N` spawns N ranks (torch.distributed.run, gloo in
--dry-run) that partition the views and reduce the step time with MAX; the reference arm runs the
reference's compiled code (oracle/_ref) or the oracle and never maps the product library."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, env=None, timeout=300):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, env=e, cwd=ROOT)
    return p


def last_json(out):
    return json.loads([ln for ln in out.strip().splitlines() if ln.startswith("{")][-1])


def test_gpus_flag_spawns_ranks_c5():
    p = run(["--dry-run", "--gpus", "2", "--workload", "c5", "--steps", "2"])
    assert p.returncode == 0, p.stderr[-2000:]
    d = last_json(p.stdout)
    assert d["n_gpus"] == 2
    views = sorted(v for r in d["ranks"] for v in r["views"])
    assert views == list(range(256))  # every trajectory view exactly once
    assert [r["views"][0] for r in sorted(d["ranks"], key=lambda r: r["rank"])] == [0, 128]


def test_gpus_flag_weak_scaling_views():
    p = run(["--dry-run", "--gpus", "2", "--workload", "c3", "--steps", "1"])
    assert p.returncode == 0, p.stderr[-2000:]
    d = last_json(p.stdout)
    ranks = sorted(d["ranks"], key=lambda r: r["rank"])
    assert [r["views"] for r in ranks] == [[0], [1]]
    assert ranks[0]["t_cw"] != ranks[1]["t_cw"]  # rank 1 renders trajectory view 1, not the street camera


def test_world_size_must_match_gpus():
    p = run(["--dry-run", "--gpus", "2"], env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert p.returncode == 2


def test_reference_arm_loads_no_product_library():
    p = run(["--impl", "reference", "--workload", "c1", "--steps", "1", "--warmup", "0"], timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    d = last_json(p.stdout)
    assert d["impl"] == "reference" and d["value"] > 0
    assert not any("libpsm" in lib for lib in d["libs_loaded"]), d["libs_loaded"]
    assert all(lib.startswith("oracle/") for lib in d["libs_loaded"]), d["libs_loaded"]
    from oracle import pyref
    assert d["cpu_baseline"]["kind"] == ("reference" if pyref.available() else "port")
