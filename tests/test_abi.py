"""The C-ABI library loads and exports every symbol include/pip.h declares;
sizing and status helpers work without a GPU (no compute calls here)."""
from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    txt = (ROOT / "include" / "pip.h").read_text()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(pip_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_header():
    from paper_2103_01216_b200 import _lib

    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    # the Python binding covers the whole header
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)


def test_library_is_sm100a():
    import subprocess

    from paper_2103_01216_b200 import _lib

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.lib_path())],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_status_strings_and_version():
    from paper_2103_01216_b200 import _lib

    lib = _lib.load()
    assert lib.pip_version() == 1
    for code in range(11):
        assert lib.pip_status_string(code)
    assert b"unsorted" in lib.pip_status_string(_lib.PIP_ERR_UNSORTED)


def test_error_mapping():
    from paper_2103_01216_b200 import _lib
    from paper_2103_01216_b200.detres import LivelockError

    with pytest.raises(ValueError):
        _lib.check(_lib.PIP_ERR_INVALID_SWAPS, "x")
    with pytest.raises(ValueError):
        _lib.check(_lib.PIP_ERR_UNSORTED, "x")
    with pytest.raises(LivelockError):
        _lib.check(_lib.PIP_ERR_LIVELOCK, "x")
    with pytest.raises(_lib.PipError):
        _lib.check(_lib.PIP_ERR_OOM, "x")


def test_workspace_sizing_is_sublinear():
    """relaxed workspace stays within 8 b(n) words for the configs' budgets
    (the acceptance gate, test_acceptance.py:257)."""
    from paper_2103_01216_b200 import _lib
    from paper_2103_01216_b200.runtime import EpsilonConfig

    lib = _lib.load()
    for n in (10**5, 10**6, 1 << 26, 1 << 30):
        b = EpsilonConfig(0.5).prefix_words(n)
        words = lib.pip_rp_workspace_bytes(n, b, 3) / 8
        assert words <= 8 * b, (n, words / b)
    for n in (1 << 20, 1 << 32):
        b = EpsilonConfig(0.5).prefix_words(n)
        words = lib.pip_merge_workspace_bytes(n, n // 2, b) / 8
        assert 0 < words <= b, (n, words / b)


def test_host_entry_points_reject_bad_predicates_before_any_transfer():
    # checked before the device is touched, so this runs without a GPU
    import numpy as np

    from paper_2103_01216_b200 import _lib

    lib = _lib.load()
    a = np.arange(10, dtype=np.uint64)
    m = C.c_uint64(0)
    for kind, pa in ((99, 0), (2, 0)):  # unknown kind; x % 0
        p = _lib.PipPred(kind, 0, pa, 0)
        assert lib.pip_filter_u64_host(a.ctypes.data, len(a), C.byref(p), C.byref(m), 0) == 1
        assert lib.pip_partition_u64_host(a.ctypes.data, len(a), C.byref(p), C.byref(m), 0) == 1
    assert np.array_equal(a, np.arange(10, dtype=np.uint64))


def test_header_compiles_as_plain_c_and_cpp(tmp_path):
    """A C or C++ binder includes pip.h on its own: no CUDA
    or torch types in the signatures."""
    import shutil
    import subprocess

    if not shutil.which("gcc"):
        pytest.skip("gcc unavailable")
    src = tmp_path / "use.c"
    src.write_text('#include "pip.h"\nint main(void) { return pip_version() == 1 ? 0 : 1; }\n')
    for cmd in (["gcc", "-std=c99", "-fsyntax-only", "-Wall", "-Werror"],
                ["g++", "-std=c++11", "-fsyntax-only", "-Wall", "-Werror", "-x", "c++"]):
        r = subprocess.run(cmd + ["-I", str(ROOT / "include"), str(src)], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
