"""The C ABI used from plain C (examples/c_api_demo.c): no Python and no torch in the
process -- the boundary a cgo / JNI / N-API binding would sit on."""

import os
import shutil
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_c_program_renders_through_the_abi(tmp_path):
    from paper_2602_03002_b200 import _native
    lib_dir = os.path.dirname(_native.LIB_PATH)
    exe = tmp_path / "c_api_demo"
    cuda = "/usr/local/cuda"
    cmd = ["gcc", "-O2", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(cuda, "include"),
           os.path.join(ROOT, "examples", "c_api_demo.c"), "-o", str(exe), "-L", lib_dir, "-l:libmdrt.so",
           "-L", os.path.join(cuda, "lib64"), "-lcudart", f"-Wl,-rpath,{lib_dir}", "-lm"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert run.returncode == 0, run.stdout + run.stderr
    assert "c_api_demo ok" in run.stdout
