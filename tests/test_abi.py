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


def test_binding_enum_values_match_the_header():
    """The Python binding's option / path / kernel constants are the header's enum values."""
    from paper_2006_10350_b200 import binding
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    enums = {k: int(v) for k, v in re.findall(r"\b(FALKON_[A-Z_0-9]+)\s*=\s*(\d+)", src)}
    pairs = {"OPT_PATH": "FALKON_OPT_PATH", "OPT_TC_MIN_D": "FALKON_OPT_TC_MIN_D",
             "OPT_TC_TERMS": "FALKON_OPT_TC_TERMS", "OPT_KERNEL_TIMING": "FALKON_OPT_KERNEL_TIMING",
             "OPT_EXP_OFFLOAD": "FALKON_OPT_EXP_OFFLOAD", "OPT_POTRF_OUTER": "FALKON_OPT_POTRF_OUTER",
             "OPT_GEMM_WARPS": "FALKON_OPT_GEMM_WARPS", "OPT_SINGLE_EVAL": "FALKON_OPT_SINGLE_EVAL",
             "OPT_STRIP_BYTES": "FALKON_OPT_STRIP_BYTES", "OPT_TC_CLUSTER": "FALKON_OPT_TC_CLUSTER",
             "OPT_LOOKAHEAD": "FALKON_OPT_LOOKAHEAD", "OPT_ACCUM_F64": "FALKON_OPT_ACCUM_F64", "OPT_DIST_PRECOND": "FALKON_OPT_DIST_PRECOND", "OPT_FIT_PRECISE": "FALKON_OPT_FIT_PRECISE", "OPT_SE_GEMV_SMS": "FALKON_OPT_SE_GEMV_SMS", "OPT_OZAKI": "FALKON_OPT_OZAKI",
             "PATH_AUTO": "FALKON_PATH_AUTO",
             "PATH_SIMT": "FALKON_PATH_SIMT", "PATH_TENSOR": "FALKON_PATH_TENSOR", "PATH_F64": "FALKON_PATH_F64",
             "GAUSSIAN": "FALKON_GAUSSIAN", "LAPLACIAN": "FALKON_LAPLACIAN"}
    for py, c in pairs.items():
        assert getattr(binding, py) == enums[c], (py, c)
    opts = {k for k in enums if k.startswith("FALKON_OPT_")}
    assert opts == {c for c in pairs.values() if c.startswith("FALKON_OPT_")}
