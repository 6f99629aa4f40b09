"""The C header is usable from plain C: compile tests/c/capi_demo.c with gcc
against include/zk_b200.h and libzk_b200.so and run it. Without a GPU the
program must see the library fail loudly (exit 77); with one, every check
passes (exit 0)."""

import os
import shutil
import subprocess

import pytest

from conftest import ROOT

from paper_2409_19156_b200 import _lib


def _build(tmp_path):
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    exe = tmp_path / "capi_demo"
    libdir = os.path.dirname(_lib.LIB_PATH)
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", os.path.join(ROOT, "tests", "c", "capi_demo.c"),
                    "-I", os.path.join(ROOT, "include"), "-L", libdir, "-lzk_b200",
                    f"-Wl,-rpath,{libdir}", "-lm", "-o", str(exe)], check=True)
    return exe


def test_c_client_builds_and_runs(tmp_path):
    exe = _build(tmp_path)
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert res.returncode in (0, 77), (res.returncode, res.stdout, res.stderr)


@pytest.mark.gpu
def test_c_client_on_gpu(tmp_path):
    exe = _build(tmp_path)
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, (res.returncode, res.stdout, res.stderr)
    assert "capi_demo ok" in res.stdout
