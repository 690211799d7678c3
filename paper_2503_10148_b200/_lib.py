"""ctypes mirror of include/sss.h and the loader of libsss.so.

Argument marshalling only: every step of the hot path runs in the CUDA
kernels of libsss.so.  There is no fallback — if the library is missing the
import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libsss.so")

SSS_OK, SSS_ERR_ARG, SSS_ERR_SHAPE, SSS_ERR_CAPACITY, SSS_ERR_CUDA = range(5)
SSS_TILE = 16
SSS_MAX_BINS = 5632
SSS_REC_FLOATS = 8
SSS_COL_FLOATS = 4
SSS_G2D_FLOATS = 10
SSS_TILE_LISTS = 2
SSS_VARIANT_POSITIVE, SSS_VARIANT_GAUSSIAN, SSS_VARIANT_LOWPASS = 1, 2, 4
SSS_BWD_NU_GRAD_PAPER = 1
SSS_BWD_RASTER_ONLY = 2
SSS_BWD_PROJECTION_ONLY = 4
SSS_BWD_GRAD_ASSIGN = 8
SSS_BWD_TARGET_U8 = 16

EXPORTS = ["sss_project", "sss_bin_sort_workspace", "sss_bin_sort", "sss_check_overflow",
           "sss_render_fwd", "sss_render_bwd_workspace", "sss_render_bwd", "sss_sghmc_step",
           "sss_image_loss_workspace", "sss_image_loss", "sss_relocate_workspace", "sss_relocate",
           "sss_status_string", "sss_last_error", "sss_launch_count", "sss_alu_peaks",
           "sss_project_bwd_range"]


class sss_camera(C.Structure):
    _fields_ = [("rot", C.c_float * 9), ("trans", C.c_float * 3), ("fx", C.c_float),
                ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float), ("width", C.c_int32),
                ("height", C.c_int32), ("z_near", C.c_float)]


class sss_params(C.Structure):
    _fields_ = [("n", C.c_int64), ("sh_degree", C.c_int32), ("variant", C.c_int32),
                ("mean", C.c_void_p), ("log_scale", C.c_void_p), ("rot", C.c_void_p),
                ("raw_nu", C.c_void_p), ("raw_opacity", C.c_void_p), ("sh", C.c_void_p),
                ("block", C.c_int64), ("block_planes", C.c_int32), ("reserved", C.c_int32)]


class sss_projected(C.Structure):
    _fields_ = [("n", C.c_int64), ("n_views", C.c_int32), ("reserved", C.c_int32),
                ("rec", C.c_void_p), ("depth", C.c_void_p), ("rect", C.c_void_p), ("col", C.c_void_p)]


class sss_bins(C.Structure):
    _fields_ = [("bin_shift", C.c_int32), ("n_views", C.c_int32), ("capacity", C.c_int64),
                ("ids", C.c_void_p), ("keys", C.c_void_p), ("ranges", C.c_void_p),
                ("totals", C.c_void_p), ("overflow", C.c_void_p), ("max_per_bin", C.c_int32),
                ("reserved", C.c_int32), ("sorted", C.c_void_p), ("n_vis", C.c_void_p),
                ("resume", C.c_void_p), ("used", C.c_void_p), ("tmask", C.c_void_p)]


class sss_frame(C.Structure):
    _fields_ = [("rgb", C.c_void_p), ("final_T", C.c_void_p), ("n_contrib", C.c_void_p),
                ("last", C.c_void_p), ("tile_list", C.c_void_p), ("tile_count", C.c_void_p),
                ("tile_cap", C.c_int32), ("reserved", C.c_int32)]


class sss_sghmc_hparams(C.Structure):
    _fields_ = [("lr", C.c_float), ("friction", C.c_float), ("noise", C.c_float),
                ("gate_k", C.c_float), ("gate_t", C.c_float), ("burn_in", C.c_int32),
                ("g_adam", C.c_int32), ("lr_scale", C.c_float), ("lr_rot", C.c_float),
                ("lr_nu", C.c_float), ("lr_opacity", C.c_float), ("lr_sh", C.c_float),
                ("beta1", C.c_float), ("beta2", C.c_float), ("adam_eps", C.c_float),
                ("grad_scale", C.c_float), ("step", C.c_int64), ("seed", C.c_uint64),
                ("eps_o", C.c_float), ("eps_sigma", C.c_float), ("mu_mode", C.c_int32),
                ("plane_begin", C.c_int32), ("plane_end", C.c_int32), ("reserved", C.c_int32),
                ("skip_if", C.c_void_p), ("step_state", C.c_void_p)]


class sss_relocate_params(C.Structure):
    _fields_ = [("threshold", C.c_float), ("cap_frac", C.c_float), ("n_max", C.c_int32),
                ("reserved", C.c_int32), ("seed", C.c_uint64), ("step", C.c_int64)]


_lib = None


def load(path: str = LIB_PATH):
    """Load libsss.so (building it first if the sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("SSS_LIB", path)  # dev: load a variant build
    if not os.path.exists(path) or os.environ.get("SSS_REBUILD"):
        from . import _build

        _build.build()
    if not os.path.exists(path):
        raise RuntimeError(f"libsss.so not found at {path}: run __graft_entry__.build()")
    lib = C.CDLL(path)
    P = C.POINTER
    st = C.c_int
    vp = C.c_void_p
    sig = {
        "sss_project": (st, [P(sss_params), P(sss_camera), C.c_int32, P(sss_projected), vp]),
        "sss_bin_sort_workspace": (C.c_size_t, [C.c_int64, C.c_int32, P(sss_camera), C.c_int32]),
        "sss_bin_sort": (st, [P(sss_projected), P(sss_camera), C.c_int32, vp, C.c_size_t,
                              P(sss_bins), vp]),
        "sss_check_overflow": (st, [P(sss_bins), vp]),
        "sss_render_fwd": (st, [P(sss_projected), P(sss_bins), P(sss_camera), C.c_int32,
                                P(C.c_float), P(sss_frame), vp]),
        "sss_render_bwd_workspace": (C.c_size_t, [C.c_int64, C.c_int32]),
        "sss_render_bwd": (st, [P(sss_params), P(sss_projected), P(sss_bins), P(sss_camera),
                                C.c_int32, P(C.c_float), P(sss_frame), vp, vp, vp,
                                P(sss_params), vp, C.c_size_t, C.c_int32, vp]),
        "sss_project_bwd_range": (st, [P(sss_params), P(sss_camera), C.c_int32, vp, C.c_size_t, P(sss_params),
                                       C.c_int64, C.c_int64, vp]),
        "sss_sghmc_step": (st, [P(sss_params), P(sss_params), P(sss_params), P(sss_params), vp,
                                P(sss_sghmc_hparams), vp]),
        "sss_image_loss_workspace": (C.c_size_t, [C.c_int32, C.c_int32, C.c_int32]),
        "sss_image_loss": (st, [vp, vp, C.c_int32, C.c_int32, C.c_int32, C.c_float, vp, vp, vp,
                                C.c_size_t, vp]),
        "sss_relocate_workspace": (C.c_size_t, [C.c_int64]),
        "sss_relocate": (st, [P(sss_params), P(sss_params), P(sss_params), vp, P(sss_relocate_params),
                              vp, vp, vp, C.c_size_t, vp]),
        "sss_status_string": (C.c_char_p, [C.c_int]),
        "sss_last_error": (C.c_char_p, []),
        "sss_launch_count": (C.c_int64, [C.c_int32]),
        "sss_alu_peaks": (C.c_int, [C.POINTER(C.c_double)]),
    }
    for name, (res, args) in sig.items():
        try:
            f = getattr(lib, name)
        except AttributeError:
            if "SSS_LIB" in os.environ:  # an older variant build (dev A/B runs) may lack newer entries
                continue
            raise
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


class SSSError(RuntimeError):
    def __init__(self, status, what=""):
        lib = load()
        msg = lib.sss_status_string(status).decode()
        detail = lib.sss_last_error().decode()
        super().__init__(f"{what}: {msg} ({detail})")
        self.status = status


def check(status, what):
    if status != SSS_OK:
        raise SSSError(status, what)
