"""The reference-side C++ shim (include/sgp_b200_shim.hpp) compiles, links libsgpx and runs the
SPEC KATs through it (GPU), or reports the missing device without a CPU fallback (CPU)."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "shim_check.cpp")
PKG = os.path.join(ROOT, "paper_1410_4984_b200")


def _build(tmp_path):
    exe = str(tmp_path / "shim_check")
    subprocess.check_call(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), SRC, "-o", exe,
                           "-L", PKG, "-lsgpx", f"-Wl,-rpath,{PKG}"])
    return exe


def test_shim_compiles_and_has_no_cpu_fallback(tmp_path):
    from paper_1410_4984_b200 import _lib

    exe = _build(tmp_path)
    if _lib.load().sgpx_device_count() > 0:
        pytest.skip("GPU visible: covered by test_shim_runs_on_gpu")
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 3 and "no CPU fallback" in r.stdout


@pytest.mark.gpu
def test_shim_runs_on_gpu(tmp_path):
    r = subprocess.run([_build(tmp_path)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
