"""B200-native hot path of Student Splatting and Scooping (arXiv 2503.10148).

Layers: CUDA kernels for sm_100a (csrc/) behind the C ABI of include/sss.h
(libsss.so), this thin torch binding (api.py), the training-step
orchestration (step.py) and the view-parallel NCCL plumbing (dist.py).
"""
from . import _lib
from .api import (  # noqa: F401
    Bins,
    Frame,
    Params,
    Projected,
    cameras_c,
    grow,
    launch_count,
    n_bins_of,
    n_planes,
    sss_bin_sort,
    sss_check_overflow,
    sss_image_loss,
    sss_project,
    sss_relocate,
    sss_render_bwd,
    sss_render_fwd,
    sss_sghmc_step,
)


def load():
    """Load libsss.so; raises if the CUDA library is missing (no fallback)."""
    return _lib.load()
