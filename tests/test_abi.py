"""The C-ABI library loads and exports every symbol include/falkon.h declares (-m "not gpu").
No compute calls: this box has no GPU."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "falkon.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(falkon_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("falkon_fit", "falkon_predict", "falkon_knm_matvec", "falkon_ctx_create"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    for name in _declared():
        assert hasattr(lib, name), name
    from paper_2006_10350_b200 import binding
    assert sorted(binding.EXPORTS) == _declared()


def test_library_symbols_are_extern_c():
    so = os.path.join(ROOT, "paper_2006_10350_b200", "libfalkon.so")
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (falkon_\w+)", out))
    assert set(_declared()) <= exported


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_2006_10350_b200", "libfalkon.so")
    r = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True)
    archs = set(re.findall(r"sm_(\d+a?)", r.stdout))
    assert archs == {"100a"}, archs


def test_strerror_and_version(lib):
    assert lib.falkon_strerror(0) == b"ok"
    assert b"invalid" in lib.falkon_strerror(1)
    assert b"sm_100a" in lib.falkon_version()


def test_invalid_arguments_fail_loudly_without_gpu(lib):
    from paper_2006_10350_b200 import binding
    h = ctypes.c_void_p()
    # world/id mismatch is rejected before any device call
    assert lib.falkon_ctx_create(ctypes.byref(h), 0, 0, 2, None) == 1
    assert lib.falkon_knm_matvec(None, None, 0, 1, None, 1, 0, 1.0, None, None) == 1
    assert b"NULL" in lib.falkon_last_error() or lib.falkon_last_error()
    with pytest.raises(binding.FalkonError):
        binding._check(1)


def test_no_cpu_fallback_when_library_missing(tmp_path):
    from paper_2006_10350_b200 import binding
    saved = binding._LIB
    binding._LIB = None
    try:
        with pytest.raises(ImportError):
            binding.load(str(tmp_path / "missing.so"))
    finally:
        binding._LIB = saved
