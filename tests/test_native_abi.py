"""The C-ABI library loads and exports every symbol include/rbws_b200.h declares (no GPU)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include/rbws_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rbws_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    import build
    build.build(verbose=False)
    return ctypes.CDLL(str(build.OUT))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "rbws_mgcg_solve" in syms and "rbws_l1roc_online" in syms
    assert len(syms) >= 20


def test_every_declared_symbol_exported(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_2311_13862_b200 import _native
    assert sorted(_native.SIGNATURES) == declared_symbols()


def test_version_and_error_without_gpu(lib):
    lib.rbws_version.restype = ctypes.c_int
    assert lib.rbws_version() == 100
    lib.rbws_last_error.restype = ctypes.c_char_p
    assert isinstance(lib.rbws_last_error(), bytes)


def test_product_never_imports_oracle():
    for p in (ROOT / "paper_2311_13862_b200").rglob("*.py"):
        src = p.read_text()
        assert "import oracle" not in src and "from oracle" not in src, p
