"""CPU-side checks of the boundary: libvtgs.so builds for sm_100a, loads without a GPU, and
exports every symbol include/vtgs.h declares (no compute calls here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "vtgs.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^VTGS_API\s+[^;(]*?\b(vtgs_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2506_02741_b200 import build
    path = build.build()
    return path


def test_header_declares_the_boundary():
    names = _declared()
    for required in ("vtgs_instantiate", "vtgs_render_fwd", "vtgs_render_bwd", "vtgs_create", "vtgs_destroy"):
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib], text=True)
    exported = set(re.findall(r"\bT (vtgs_\w+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, f"declared but not exported: {missing}"
    # nothing but the C ABI leaks out
    assert all(n.startswith("vtgs_") for n in exported)


def test_binding_names_match_header(lib):
    from paper_2506_02741_b200 import vtgs
    assert sorted(vtgs.EXPORTED) == _declared()
    assert vtgs.vtgs_abi_version() == 4
    for s in (0, -1, -2, -3, -4, -5, -6):
        assert vtgs.vtgs_status_string(s)


def test_sass_is_sm100a(lib):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib], text=True)
    assert "sm_100a" in out


def test_no_device_means_error_not_fallback(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2506_02741_b200 import vtgs
    h = ctypes.c_void_p()
    assert vtgs.vtgs_create(ctypes.byref(h), 0, 16, 16, 16, 0) == vtgs.VTGS_ERR_NO_DEVICE
    with pytest.raises(vtgs.VtgsError):
        vtgs.Renderer(0, 16, 16, 16)


def test_product_does_not_import_oracle():
    """The product package never imports the oracle (task rule ③)."""
    pkg = os.path.join(ROOT, "paper_2506_02741_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", src, flags=re.M), f
                assert "vtgs_oracle" not in src and "oracle_impl" not in src, f
