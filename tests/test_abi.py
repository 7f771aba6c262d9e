"""The C ABI library: loads without a GPU, exports every symbol include/mdrt.h
declares, and the ctypes structure layouts match the C header (checked by
compiling a probe against the header with gcc)."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2602_03002_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mdrt.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mdrt_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_expected_entry_points():
    names = declared_functions()
    assert "mdrt_render" in names and "mdrt_create" in names and "mdrt_last_error" in names
    assert sorted(_native.EXPORTS) == names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_abi_version_and_errors_without_gpu():
    L = _native.lib()
    assert L.mdrt_abi_version() == _native.ABI_VERSION == 2
    n = _native.device_count()
    assert n >= 0
    if n == 0:
        ptr = ctypes.c_void_p()
        rc = L.mdrt_create(0, ctypes.byref(ptr))
        assert rc != 0
        assert L.mdrt_last_error()          # message set
    # argument errors map to ValueError (reference error behaviour)
    with pytest.raises(ValueError):
        _native.check(L.mdrt_render(None, None, None))


def _c_layout(struct, fields):
    src = ['#include <stddef.h>', '#include <stdio.h>', f'#include "{HEADER}"', "int main(void) {",
           f'  printf("%zu\\n", sizeof({struct}));']
    src += [f'  printf("%zu\\n", offsetof({struct}, {f}));' for f in fields]
    src += ["  return 0;", "}"]
    d = os.path.join(ROOT, "build")
    os.makedirs(d, exist_ok=True)
    c = os.path.join(d, f"layout_{struct}.c")
    exe = c[:-2]
    open(c, "w").write("\n".join(src))
    subprocess.run(["gcc", "-std=c11", c, "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()
    return int(out[0]), [int(x) for x in out[1:]]


@pytest.mark.parametrize("cls,cname", [(_native.StepArgs, "mdrt_step_args"), (_native.Stats, "mdrt_stats")])
def test_ctypes_struct_layout_matches_header(cls, cname):
    fields = [f for f, _ in cls._fields_]
    size, offs = _c_layout(cname, fields)
    assert ctypes.sizeof(cls) == size
    assert [getattr(cls, f).offset for f in fields] == offs


def test_host_touch_and_copy_cpu():
    """mdrt_host_touch leaves values unchanged; mdrt_host_copy equals memcpy for any size and
    thread count (4 KB-aligned slices, the persistent host pool)."""
    import numpy as np
    from paper_2602_03002_b200 import _native
    L = _native.lib()
    rng = np.random.default_rng(0)
    for size in (0, 1, 4095, 4096, 4097, 3 * 4096 + 5, (10 << 20) + 123):
        src = rng.integers(0, 255, size=max(size, 1), dtype=np.uint8)[:size]
        for th in (1, 3, 8, 16):
            dst = np.zeros(max(size, 1), np.uint8)[:size]
            assert L.mdrt_host_copy(dst.ctypes.data, src.ctypes.data, size, th) == 0
            assert np.array_equal(dst, src)
            keep = dst.copy()
            assert L.mdrt_host_touch(dst.ctypes.data, size, th) == 0
            assert np.array_equal(dst, keep)
    assert L.mdrt_host_copy(None, None, 16, 1) == _native.MDRT_EINVAL
    assert L.mdrt_host_touch(None, 16, 0) == _native.MDRT_EINVAL
