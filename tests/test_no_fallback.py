"""The product path never routes through the oracle or a CPU fallback.

Static checks over the shipped package (`paper_2602_03002_b200/`): no module
imports or loads anything under `oracle/`, and the native loader raises when
libmdrt.so is absent instead of degrading to Python/numpy.
"""
import ast
import pathlib

import pytest

PKG = pathlib.Path(__file__).resolve().parents[1] / "paper_2602_03002_b200"


def _py_files():
    return sorted(p for p in PKG.rglob("*.py") if "__pycache__" not in p.parts)


@pytest.mark.parametrize("path", _py_files(), ids=lambda p: str(p.relative_to(PKG)))
def test_package_does_not_import_oracle(path):
    tree = ast.parse(path.read_text(), filename=str(path))
    for node in ast.walk(tree):
        if isinstance(node, ast.Import):
            names = [a.name for a in node.names]
        elif isinstance(node, ast.ImportFrom):
            names = [node.module or ""]
        else:
            continue
        for n in names:
            assert not n.split(".")[0] == "oracle", f"{path}: imports {n}"
    src = path.read_text()
    assert "liboracle" not in src and "oracle/_ref" not in src, f"{path} references the oracle library"


def test_loader_raises_without_library(tmp_path, monkeypatch):
    from paper_2602_03002_b200 import _native

    monkeypatch.setattr(_native, "LIB_PATH", str(tmp_path / "missing_libmdrt.so"), raising=False)
    for attr in ("_LIB", "_lib"):
        if hasattr(_native, attr):
            monkeypatch.setattr(_native, attr, None)
    loader = getattr(_native, "lib", None) or getattr(_native, "load", None)
    if loader is None:
        pytest.skip("no loader entry point exposed")
    with pytest.raises((ImportError, OSError)):
        loader()
