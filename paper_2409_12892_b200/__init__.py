"""splatlm-b200: B200-native (sm_100a) 3DGS-LM inner solver.

Drop-in for the reference `splatlm` hot path (cache build -> PCG -> Eq. 7
combine); see DESIGN.md.  Public API mirrors the reference module layout:

    scene:      GaussianScene, Camera, ParamVector, Layout, sort_x, sort_x_inverse,
                flatten, unflatten, scene_with_offset, JSON IO
    rasterizer: RenderConfig, project_scene, render
    residuals:  compute_residuals, ResidualBundle
    jacobian:   build_cache, sort_cache_by_gaussians, apply_j, weight_residuals,
                apply_jt, diag_jtj, dump_cache, load_cache_dump
    solver:     pcg_solve, solve_normal_equations_batched, lm_direction
    lm:         line_search, compute_rho, trust_region_update, lm_step
    fit:        adam_fit, lm_fit, two_stage_fit (SPEC-only drivers); CLI: python -m paper_2409_12892_b200
"""

from .errors import CacheOrderError, ImageSizeError, LayoutError, NonSPDError, SplatLMError  # noqa: F401
from .scene import (Camera, GaussianScene, Layout, ParamVector, flatten, scene_with_offset,  # noqa: F401
                    sort_x, sort_x_inverse, unflatten)

__all__ = ["Camera", "GaussianScene", "Layout", "ParamVector", "flatten", "unflatten", "sort_x",
           "sort_x_inverse", "scene_with_offset", "CacheOrderError", "ImageSizeError", "LayoutError",
           "NonSPDError", "SplatLMError"]
