"""The C-ABI library builds, loads without a GPU, exports exactly what include/readme.h declares, and
rejects bad arguments synchronously (no compute call is made here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "readme.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(readme_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2410_19123_b200 import build, readme
    build.build()
    return readme.lib()


def test_header_symbols_exported(lib):
    from paper_2410_19123_b200 import readme
    so = readme.LIB_PATH
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True, check=True).stdout
    exported = sorted(set(re.findall(r" T (readme_\w+)", out)))
    assert exported == _declared()
    assert sorted(readme.EXPORTS) == _declared()
    for name in _declared():
        assert hasattr(lib, name)


def test_no_internal_symbols_leak():
    from paper_2410_19123_b200 import readme
    out = subprocess.run(["nm", "-D", "--defined-only", readme.LIB_PATH], capture_output=True, text=True).stdout
    assert not re.search(r" T _ZN6readme", out)


def test_version_and_strings(lib):
    assert lib.readme_version() == 1
    assert lib.readme_status_string(0) == b"README_OK"
    assert lib.readme_status_string(3) == b"README_ERR_WORKSPACE"


def test_workspace_sizes(lib):
    assert lib.readme_route_workspace_bytes(8192, 8, 1) >= 32 * 8 * 8
    assert lib.readme_expert_ffn_workspace_bytes(8192, 4096, 8, 5504, 1) >= 8192 * 5504 * 2
    w = lib.readme_moe_layer_workspace_bytes(8192, 4096, 8, 5504, 1, 1)
    assert w >= 2 * 8192 * 4096 * 2 + 8192 * 5504 * 2


@pytest.mark.parametrize("T,E,k,msg", [(-1, 8, 1, b"T must"), (10, 0, 1, b"E must"), (10, 300, 1, b"E must"),
                                       (10, 8, 9, b"k must"), (10, 8, 0, b"k must")])
def test_route_rejects_bad_args(lib, T, E, k, msg):
    dummy = ctypes.c_void_p(16)
    rc = lib.readme_route(dummy, 0, T, E, k, dummy, dummy, dummy, dummy, dummy, None, None, dummy, 1 << 20, None)
    assert rc == 1 and msg in lib.readme_last_error()


def test_route_workspace_too_small(lib):
    dummy = ctypes.c_void_p(16)
    rc = lib.readme_route(dummy, 0, 4096, 8, 1, dummy, dummy, dummy, dummy, dummy, None, None, dummy, 8, None)
    assert rc == 3


def test_ffn_rejects_bad_shapes(lib):
    d = ctypes.c_void_p(16)
    # H not a multiple of 8
    assert lib.readme_expert_ffn(d, 1, 10, 12, 8, 64, 1, d, d, d, d, d, None, d, 1 << 30, None) == 1
    # d not a multiple of 8
    assert lib.readme_expert_ffn(d, 1, 10, 64, 8, 60, 1, d, d, d, d, d, None, d, 1 << 30, None) == 1
    # unknown dtype
    assert lib.readme_expert_ffn(d, 7, 10, 64, 8, 64, 1, d, d, d, d, d, None, d, 1 << 30, None) == 2
    # misaligned pointer
    assert lib.readme_expert_ffn(ctypes.c_void_p(18), 1, 10, 64, 8, 64, 1, d, d, d, d, d, None, d, 1 << 30, None) == 1


def test_no_cpu_fallback_in_binding():
    import torch
    from paper_2410_19123_b200 import readme
    with pytest.raises(ValueError, match="CUDA"):
        readme.route(torch.zeros(4, 8), 1)


def test_knobs_set_get_reset(lib):
    """Lab switches: read once from the environment, overridable, unknown names rejected synchronously."""
    v = ctypes.c_int32(-99)
    assert lib.readme_debug_get_knob(b"ffn_mt", ctypes.byref(v)) == 0 and v.value == 0
    assert lib.readme_debug_set_knob(b"ffn_mt", 128) == 0
    assert lib.readme_debug_get_knob(b"ffn_mt", ctypes.byref(v)) == 0 and v.value == 128
    assert lib.readme_debug_reset_knob(b"ffn_mt") == 0
    assert lib.readme_debug_get_knob(b"ffn_mt", ctypes.byref(v)) == 0 and v.value == 0
    assert lib.readme_debug_set_knob(b"no_such_knob", 1) == 1
    assert b"unknown knob" in lib.readme_last_error()
    assert lib.readme_debug_get_knob(b"ffn_spin", ctypes.byref(v)) == 0 and v.value == 25
