"""Bounds-checked build (MDRT_CHECKS): the GPU parity suite re-run against
libmdrt_checked.so, where every node, triangle, stack, pixel, ring-slot and
downsample index is checked on the device before it is used, plus a
corrupted tree that must trip the stack check instead of running off the end
of the traversal stack.

The checked library is loaded through MDRT_LIB in a child process, so this
process keeps the release build.
"""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = ["tests/test_gpu_parity.py", "tests/test_gpu_edge.py", "tests/test_gpu_api.py",
         "tests/test_gpu_acceptance.py", "tests/test_bvh_api.py", "tests/test_gpu_entry.py",
         "tests/test_gpu_lifetime.py", "tests/test_gpu_seam.py"]

pytestmark = pytest.mark.skipif(os.environ.get("MDRT_CHECKED_CHILD") == "1",
                                reason="already running under the checked build")


def _checked_env():
    from paper_2602_03002_b200 import build
    lib = build.build_checked()
    env = dict(os.environ, MDRT_LIB=lib, MDRT_CHECKED_CHILD="1")
    return lib, env


@pytest.mark.gpu
def test_gpu_suite_under_bounds_checks():
    lib, env = _checked_env()
    suite = [s for s in SUITE if os.path.exists(os.path.join(ROOT, s))]
    res = subprocess.run([sys.executable, "-m", "pytest", *suite, "-m", "gpu", "-x", "-q", "-p", "no:cacheprovider",
                          "-k", "not sm_local_tile_schedule"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    tail = (res.stdout + res.stderr)[-4000:]
    assert "MDRT_CHECK" not in res.stdout + res.stderr, tail
    assert res.returncode == 0, tail
    import re
    m = re.search(r"(\d+) passed", res.stdout)
    assert m and int(m.group(1)) >= 40, tail   # the parity suite ran, not a skipped shell


_CYCLE = r"""
import ctypes, sys, numpy as np, torch
from paper_2602_03002_b200 import _native
assert _native.LIB_PATH.endswith("libmdrt_checked.so"), _native.LIB_PATH
# one inner record whose children are both itself, with boxes around everything:
# every ray descends into node 0 forever, pushing a stack entry per visit
node = np.zeros(16, np.float32)
big = [-10.0, 10.0, -10.0, 10.0]
node[0:4] = big; node[4:8] = big          # child 0 x/y, child 1 x/y
node[8:12] = [-10.0, 10.0, -10.0, 10.0]   # child 0 z, child 1 z
node[12:14] = np.array([0, 0], np.int32).view(np.float32)
nodes = torch.from_numpy(node).cuda()
tris = torch.zeros(12, device="cuda")
o = torch.zeros(3, device="cuda"); d = torch.tensor([1.0, 0.5, 0.25], device="cuda")
t = torch.empty(1, device="cuda"); f = torch.empty(1, dtype=torch.int32, device="cuda")
rc = _native.lib().mdrt_query_rays(ctypes.c_void_p(nodes.data_ptr()), ctypes.c_void_p(tris.data_ptr()),
    ctypes.c_void_p(o.data_ptr()), ctypes.c_void_p(d.data_ptr()), 1, 100.0, ctypes.c_void_p(t.data_ptr()),
    ctypes.c_void_p(f.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
print("NOT TRAPPED", rc)
"""


@pytest.mark.gpu
def test_corrupted_tree_trips_stack_check():
    _, env = _checked_env()
    res = subprocess.run([sys.executable, "-c", _CYCLE], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=300)
    out = res.stdout + res.stderr
    assert "NOT TRAPPED" not in out, out[-2000:]
    assert res.returncode != 0
    assert "MDRT_CHECK" in out and "stack depth" in out, out[-2000:]
