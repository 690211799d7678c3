"""CPU checks of the C-ABI library: it builds for sm_100a, loads, exports every
symbol include/sss.h declares, and validates arguments synchronously (no GPU
needed: validation returns before any CUDA call)."""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT


@pytest.fixture(scope="module")
def lib():
    from paper_2503_10148_b200 import _build, _lib

    _build.build()
    return _lib.load()


def _declared():
    src = open(os.path.join(ROOT, "include", "sss.h")).read()
    return sorted(set(re.findall(r"SSS_API\s+[\w\s\*]+?\b(sss_\w+)\s*\(", src)))


def test_header_declares_the_five_hot_path_calls():
    names = _declared()
    for k in ["sss_project", "sss_bin_sort", "sss_render_fwd", "sss_render_bwd", "sss_sghmc_step"]:
        assert k in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2503_10148_b200 import _lib

    names = _declared()
    assert len(names) >= 11
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(_lib.EXPORTS) == names


def test_library_is_sm100a(lib):
    import subprocess

    from paper_2503_10148_b200._lib import LIB_PATH

    out = subprocess.run(["cuobjdump", "--list-elf", LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_argument_validation_is_synchronous(lib):
    from paper_2503_10148_b200 import _lib as L

    assert lib.sss_status_string(L.SSS_ERR_ARG).decode().startswith("SSS_ERR_ARG")
    cam = L.sss_camera()
    cam.fx = cam.fy = 100.0
    cam.width, cam.height, cam.z_near = 64, 64, 0.2
    p = L.sss_params(10, 5, 0, None, None, None, None, None, None)  # bad degree
    out = L.sss_projected(10, 1, 0, None, None, None)
    assert lib.sss_project(C.byref(p), C.byref(cam), 1, C.byref(out), None) == L.SSS_ERR_ARG
    assert b"sh_degree" in lib.sss_last_error()
    p = L.sss_params(-1, 0, 0, None, None, None, None, None, None)
    assert lib.sss_project(C.byref(p), C.byref(cam), 1, C.byref(out), None) == L.SSS_ERR_ARG
    p = L.sss_params(0, 0, 0, None, None, None, None, None, None)
    bad = L.sss_camera()
    bad.fx = bad.fy = 1.0
    bad.width, bad.height, bad.z_near = 0, 10, 0.2
    out0 = L.sss_projected(0, 1, 0, None, None, None)
    assert lib.sss_project(C.byref(p), C.byref(bad), 1, C.byref(out0), None) == L.SSS_ERR_SHAPE
    bad.width, bad.fx = 10, -1.0
    assert lib.sss_project(C.byref(p), C.byref(bad), 1, C.byref(out0), None) == L.SSS_ERR_ARG
    two = (L.sss_camera * 2)(cam, cam)
    two[1].width = 32
    out2 = L.sss_projected(0, 2, 0, None, None, None)
    assert lib.sss_project(C.byref(p), two, 2, C.byref(out2), None) == L.SSS_ERR_SHAPE
    # the scatter packs bin coordinates in 10 bits: > 1024 bins per axis is a shape error
    wide = L.sss_camera()
    wide.fx = wide.fy = 100.0
    wide.width, wide.height, wide.z_near = 16 * 1025, 16, 0.2
    prw = L.sss_projected(0, 1, 0, None, None, None)
    bw = L.sss_bins(0, 1, 0, None, None, None, None, None)
    assert lib.sss_bin_sort(C.byref(prw), C.byref(wide), 1, None, 0, C.byref(bw), None) == L.SSS_ERR_SHAPE
    assert b"1024 per axis" in lib.sss_last_error()
    assert lib.sss_bin_sort_workspace(-1, 1, C.byref(cam), 0) == 0
    assert lib.sss_bin_sort_workspace(1000, 1, C.byref(cam), 0) > 0
    assert lib.sss_render_bwd_workspace(1000, 2) == 1000 * 2 * L.SSS_G2D_FLOATS * 4 == 80000
    h = L.sss_sghmc_hparams()
    pp = L.sss_params(0, 0, 0, None, None, None, None, None, None)
    assert lib.sss_sghmc_step(C.byref(pp), C.byref(pp), C.byref(pp), C.byref(pp), None,
                              C.byref(h), None) == L.SSS_ERR_ARG  # step 0 / lr 0


def test_product_never_imports_the_oracle():
    """The CUDA path has no CPU fallback and shares nothing with oracle/."""
    pkg = os.path.join(ROOT, "paper_2503_10148_b200")
    pat = re.compile(r"(import\s+oracle|from\s+oracle|liboracle|sss_oracle|orc_)")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not pat.search(txt), f
