"""Build libmdrt.so in-tree with nvcc for sm_100a (no JIT, no torch extension cache).

    python -m paper_2602_03002_b200.build [--verbose]

The shared library lands next to this file so it travels with the repo
snapshot to GPU boxes; it is git-ignored (*.so).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libmdrt.so")
# diagnostic variant with device-side bounds checks (MDRT_CHECKS): load it with
# MDRT_LIB=<path> to run any test or tool with every index checked
LIB_CHECKED = os.path.join(HERE, "libmdrt_checked.so")
SOURCES = ["bvh_build.cpp", "mdrt_kernels.cu", "mdrt_api.cu"]
HEADERS = ["bvh_build.h", "mdrt_device.cuh", "mdrt_kernels.h"]

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libmdrt.so")


def _inputs() -> list[str]:
    files = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    files.append(os.path.join(ROOT, "include", "mdrt.h"))
    files.append(os.path.abspath(__file__))
    return files


def up_to_date(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(f) <= t for f in _inputs())


def build_checked(force: bool = False) -> str:
    """Compile libmdrt_checked.so (MDRT_CHECKS) unless it is up to date."""
    if not force and up_to_date(LIB_CHECKED):
        return LIB_CHECKED
    return build(out=LIB_CHECKED, defines=("MDRT_CHECKS",))


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple[str, ...] = ()) -> str:
    """Compile libmdrt.so; ``out``/``defines`` produce kernel variants for experiments."""
    target = out or LIB
    if not force and out is None and not defines and up_to_date():
        return LIB
    cmd = [nvcc_path(), *ARCH_FLAGS, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
           "-shared", "-cudart", "static", "-I", os.path.join(ROOT, "include"),
           *[f"-D{d}" for d in defines],
           *[os.path.join(CSRC, f) for f in SOURCES], "-o", target + ".tmp"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--out", default=None)
    ap.add_argument("-D", dest="defines", action="append", default=[])
    ap.add_argument("--checked", action="store_true", help="build libmdrt_checked.so (MDRT_CHECKS)")
    a = ap.parse_args()
    if a.checked:
        print(build_checked(force=a.force))
    else:
        print(build(force=a.force, verbose=a.verbose, out=a.out, defines=tuple(a.defines)))
