"""Builds the C++ drop-in shim tests and runs them on the GPU: tests/cpp/test_raster_b200.cpp (a port
of the render cases of proj/tests/test_raster.cpp over include/psimap_b200.hpp) and
tests/cpp/acceptance_b200.cpp (the reference's acceptance criteria 1-3, acceptance.cpp:45-167, through
the shim's stage functions, RenderCache and bench_render)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2604_10982_b200")


def _build(tmp_path, name="test_raster_b200"):
    exe = str(tmp_path / name)
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", name + ".cpp"), "-L", LIBDIR, "-lpsm",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_cpp_shim_compiles(tmp_path):
    assert os.path.exists(_build(tmp_path))
    assert os.path.exists(_build(tmp_path, "acceptance_b200"))


@pytest.mark.gpu
def test_cpp_shim_render_cases(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_acceptance_criteria_1_to_3(tmp_path):
    exe = _build(tmp_path, "acceptance_b200")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
