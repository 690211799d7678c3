"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds *only* input generation (component parameters, cameras,
target images, optimiser hyper-parameters).  It contains none of the method's
arithmetic (no projection, compositing, gradients or sampler maths), so both
`oracle/` and `paper_2503_10148_b200/` may consume it without sharing code.
"""
from .scenes import (  # noqa: F401
    Camera,
    Scene,
    SGHMCParams,
    CONFIG_NAMES,
    make_scene,
    make_custom_scene,
    make_stress_scene,
    make_stop_rule_scene,
    make_optimizer_state,
    sghmc_params_for,
    make_targets,
    make_targets_u8,
    make_cameras,
    look_at,
    sh_coeff_count,
    param_plane_count,
)
