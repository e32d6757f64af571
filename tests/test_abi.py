"""CPU-side checks of the C ABI library: it loads and exports every symbol that
``include/paraexp.h`` declares; without a GPU it reports errors instead of crashing.
No compute calls here (no GPU in the CPU suite)."""

import ctypes
import os
import re

import pytest

from tests.conftest import ROOT

HEADER = os.path.join(ROOT, "include", "paraexp.h")


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(px_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2004_00546_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return _native.load()


def test_header_declares_expected_api():
    names = declared_functions()
    for n in ("px_create", "px_destroy", "px_direct", "px_adjoint", "px_gradient", "px_get", "px_set_cheb_plan"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    raw = ctypes.CDLL(os.path.join(ROOT, "paper_2004_00546_b200", "libparaexp.so"))
    missing = [n for n in declared_functions() if not hasattr(raw, n)]
    assert not missing, missing


def test_bindings_cover_the_header(lib):
    from paper_2004_00546_b200._native import SIGNATURES
    assert set(declared_functions()) == set(SIGNATURES)


def test_abi_version_and_build_info(lib):
    from paper_2004_00546_b200 import _native as N
    assert lib.px_abi_version() == N.ABI_VERSION == 5
    assert b"sm_100a" in lib.px_build_info()


def test_create_rejects_bad_descriptor_without_crashing(lib):
    from paper_2004_00546_b200 import _native as N
    d = N.ProblemDesc()
    d.nx = 2  # invalid grid
    h = ctypes.c_void_p()
    rc = lib.px_create(ctypes.byref(d), ctypes.byref(h))
    assert rc == 1  # PX_ERR_ARG
    assert b"grid" in lib.px_last_error(None)


def test_struct_layouts_match_header(lib):
    from paper_2004_00546_b200 import _native as N
    # px_problem_desc: 3 ints, pad, 5 doubles, 3 doubles, 12 ints
    assert ctypes.sizeof(N.ProblemDesc) == 16 + 40 + 24 + 48
    assert ctypes.sizeof(N.ChebPlanC) == 8 + 4 + 4 + 8 + 8 + 8 + 8 + 8
    assert ctypes.sizeof(N.Stats) == 4 * 8 + 3 * 8


def test_no_cpu_fallback_when_library_missing(tmp_path, monkeypatch):
    from paper_2004_00546_b200 import _native as N
    from paper_2004_00546_b200.errors import NativeUnavailable
    with pytest.raises(NativeUnavailable):
        N.load(str(tmp_path / "missing.so"))


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2004_00546_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, flags=re.M), f
