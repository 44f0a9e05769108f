"""On-disk boundary of the render path: checkpoints, raw planes,
PPM, camera JSON and bench reports (proj/src/io.cpp), in C++ (include/psimap_b200_io.hpp,
tests/cpp/test_io_b200.cpp = the render-path cases of proj/tests/test_io.cpp) and Python
(paper_2604_10982_b200/io.py), byte-compatible; and the CLI (tools/psimap_b200.cpp,
psimap_main.cpp's render / bench) driving the GPU path from those files."""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_2604_10982_b200 import (Camera, RasterConfig, SceneMap, StreetSpec, make_street_scene, street_f_ins,
                                   street_queries)
from paper_2604_10982_b200 import io as pio

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2604_10982_b200")
CLI = os.path.join(LIBDIR, "psimap_b200")


def _build_io_test(tmp_path):
    exe = str(tmp_path / "test_io_b200")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_io_b200.cpp"), "-L", LIBDIR, "-lpsm",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_cpp_io_cases(tmp_path):
    exe = _build_io_test(tmp_path)
    r = subprocess.run([exe, str(tmp_path), str(tmp_path / "fixed.psimap")], capture_output=True, text=True)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


def test_python_checkpoint_is_byte_compatible_with_cpp(tmp_path):
    exe = _build_io_test(tmp_path)
    subprocess.run([exe, str(tmp_path), str(tmp_path / "fixed.psimap")], check=True, capture_output=True)
    ck = pio.load_checkpoint(str(tmp_path / "fixed.psimap"))
    assert len(ck.scene) == 9 and ck.vocabulary == ["floor", "crate"]
    assert ck.scene.f_sem.shape == (9, 2) and ck.scene.f_ins.shape == (9, 3)
    assert [q.alive for q in ck.scene.queries] == [True, False, True]
    assert ck.class_votes == [[3, 1]] * 3 and ck.assign_count == [17, 18, 19] and ck.pos_enc_seed == 21
    pio.save_checkpoint(str(tmp_path / "py.psimap"), ck)
    assert (tmp_path / "py.psimap").read_bytes() == (tmp_path / "fixed.psimap").read_bytes()


def test_python_raw_planes_and_errors(tmp_path):
    a = np.random.default_rng(1).standard_normal((4, 6, 5))
    pio.save_raw(str(tmp_path / "f.raw"), a)
    assert np.array_equal(pio.load_raw(str(tmp_path / "f.raw")), a)
    i = np.arange(9, dtype=np.int32).reshape(3, 3, 1) - 4
    pio.save_raw(str(tmp_path / "i.raw"), i)
    back = pio.load_raw(str(tmp_path / "i.raw"))
    assert back.dtype == np.int32 and np.array_equal(back, i)
    (tmp_path / "bad.raw").write_bytes(b"NOTPLANE" + b"\0" * 16)
    with pytest.raises(RuntimeError):
        pio.load_raw(str(tmp_path / "bad.raw"))
    with pytest.raises(RuntimeError):
        pio.load_checkpoint(str(tmp_path / "f.raw"))


def test_python_camera_json_round_trip():
    cam = Camera.look_at((1, 2, 3), (0, 0, 0), (0, 1, 0), 80, 80, 64, 48, 0.1, 50.0)
    back = pio.camera_from_json(pio.camera_to_json(cam))
    assert np.max(np.abs(back.r_cw - cam.r_cw)) < 1e-14 and np.max(np.abs(back.t_cw - cam.t_cw)) < 1e-14
    la = pio.camera_from_json(json.dumps({"eye": [1, 2, 3], "target": [0, 0, 0], "up": [0, 1, 0], "fx": 80, "fy": 80,
                                          "width": 64, "height": 48, "near": 0.1, "far": 50.0}))
    assert np.max(np.abs(la.r_cw - cam.r_cw)) < 1e-12


@pytest.fixture(scope="module")
def street_ckpt(tmp_path_factory):
    d = tmp_path_factory.mktemp("street")
    spec = StreetSpec(n_surfels=12000, image_w=256, image_h=192, c_sem=16, seed=7)
    scene, _, cam = make_street_scene(spec, with_labels=False)
    sc = SceneMap(scene.surfels, scene.f_sem, street_f_ins(spec), street_queries(12))
    pio.save_checkpoint(str(d / "street.psimap"), pio.Checkpoint(sc, ["street"]))
    (d / "cam.json").write_text(pio.camera_to_json(cam))
    return d, sc, cam


def test_cli_builds():
    assert os.path.exists(CLI), "built by paper_2604_10982_b200/csrc/Makefile"


@pytest.mark.gpu
def test_cli_render_matches_oracle(street_ckpt):
    from oracle import pyoracle as O
    d, sc, cam = street_ckpt
    out = d / "render"
    r = subprocess.run([CLI, "render", "--checkpoint", str(d / "street.psimap"), "--camera", str(d / "cam.json"),
                        "--out", str(out), "--blending", "topk", "--topk", "8"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    o = O.render_panoptic(sc, sc.f_ins, sc.queries, cam, RasterConfig(blending=1, top_k=8))
    for name, key in (("color", "color"), ("depth", "depth"), ("normal", "normal"), ("sem_feat", "sem_feat"),
                      ("ins_dist", "ins_dist"), ("alpha", "alpha_acc")):
        a = pio.load_raw(str(out / f"{name}.raw"))
        assert a.shape == o[key].shape and np.max(np.abs(a - o[key])) <= 1e-4, name
    # labels blend in fp64 in blend order on the GPU (raster.cpp:486-498): the argmax is exact
    assert np.array_equal(pio.load_raw(str(out / "ins_argmax.raw"))[..., 0], o["ins_argmax"][..., 0])
    assert (out / "color.ppm").exists() and json.loads((out / "run_config.json").read_text())["topk"] == "8"


@pytest.mark.gpu
def test_cli_panoptic_bit_exact(street_ckpt):
    from oracle import pyoracle as O
    d, sc, cam = street_ckpt
    out = d / "pan"
    r = subprocess.run([CLI, "panoptic", "--checkpoint", str(d / "street.psimap"), "--camera", str(d / "cam.json"),
                        "--out", str(out), "--binning", "ellipse", "--blending", "topk", "--topk", "16"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    o = O.render_panoptic(sc, sc.f_ins, sc.queries, cam, RasterConfig(blending=1, top_k=16))
    for name in ("ids", "classes", "sem_classes"):
        assert np.array_equal(pio.load_raw(str(out / f"{name}.raw")), o[name]), name


@pytest.mark.gpu
def test_cli_bench_street(tmp_path):
    r = subprocess.run([CLI, "bench", "--street", "--street-surfels", "12000", "--reps", "2", "--out", str(tmp_path)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rep = json.loads((tmp_path / "bench.json").read_text())
    names = [row["config"] for row in rep["rows"]]
    assert names == ["baseline", "precise_tile", "topk", "full_method"]
    assert rep["rows"][2]["blended_total"] == rep["rows"][3]["blended_total"]  # acceptance.cpp:155-166
    assert (tmp_path / "bench.csv").read_text().startswith("config,binning,blending")
