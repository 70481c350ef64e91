"""ctypes binding of libsplatlm_b200.so (C ABI in include/splatlm_b200.h).

There is no fallback: importing the product path without the built library
raises.  Status codes map to the reference's exception classes.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import torch

from .errors import CacheOrderError, ImageSizeError, LayoutError, SplatLMError

_HERE = Path(__file__).resolve().parent
# SLM_LIB overrides the library path (A/B builds of tuning variants)
LIB_PATH = Path(os.environ["SLM_LIB"]) if os.environ.get("SLM_LIB") else _HERE / "libsplatlm_b200.so"

c_vp = C.c_void_p
c_ll = C.c_longlong
c_i = C.c_int
c_d = C.c_double
c_f = C.c_float


class SlmCamera(C.Structure):
    _fields_ = [("R", c_d * 9), ("t", c_d * 3), ("fx", c_d), ("fy", c_d), ("cx", c_d), ("cy", c_d),
                ("C", c_d * 3), ("W", c_i), ("H", c_i), ("pix_base", c_ll)]


class SlmRastCfg(C.Structure):
    _fields_ = [("alpha_min", c_d), ("t_stop", c_d), ("alpha_clamp", c_d), ("cov_eps", c_d),
                ("z_near", c_d), ("cull_sigma", c_d), ("reach_fac", c_d), ("bg", c_d * 3)]


class SlmView(C.Structure):
    _fields_ = [("pix_base", c_ll), ("W", c_i), ("H", c_i)]


class SlmRasterArgs(C.Structure):
    _fields_ = [("tile_range", c_vp), ("inst_gid", c_vp), ("splats", c_vp),
                ("W", c_i), ("H", c_i), ("tiles_x", c_i), ("pix_base", c_ll), ("cfg", SlmRastCfg),
                ("px_count", c_vp), ("rgb", c_vp), ("t_final", c_vp), ("inst_mask", c_vp),
                ("inst_start", c_vp), ("rec4", c_vp), ("rec_d2", c_vp), ("rec_pix", c_vp),
                ("pix_off", c_vp), ("view_entry_base", c_ll), ("trav_gid", c_vp), ("trav_alpha", c_vp),
                ("trav_T", c_vp), ("views", c_vp), ("view_tile_base", c_vp), ("n_views", c_i), ("n_tiles", c_i),
                ("rec4_h", c_vp), ("rec_d2_h", c_vp), ("rec_pix_h", c_vp), ("e_split", c_ll), ("e_hbase", c_ll)]


class SlmResidArgs(C.Structure):
    _fields_ = [("img", c_vp), ("gt", c_vp), ("gt_f32", c_i), ("W", c_i), ("H", c_i),
                ("lambda1", c_d), ("lambda2", c_d), ("eps_den", c_d), ("ssim_c1", c_d), ("ssim_c2", c_d),
                ("mode", c_i), ("win", c_i), ("taps", c_vp), ("cw_y", c_vp), ("cw_x", c_vp),
                ("gradr", c_vp), ("cgrad", c_vp), ("energy_part", c_vp),
                ("o_gradr", c_vp), ("o_cgrad", c_vp), ("o_rabs", c_vp), ("o_rssim", c_vp),
                ("o_drabs", c_vp), ("o_drssim", c_vp)]


class SlmTileArgs(C.Structure):
    _fields_ = [("views", c_vp), ("view_tile_base", c_vp), ("n_views", c_i), ("n_tiles", c_i),
                ("tile_run_off", c_vp), ("tile_chunk_off", c_vp), ("chunk_run", c_vp), ("chunk_perm", c_vp), ("run_slot", c_vp),
                ("run_start", c_vp), ("run_fn", c_vp), ("run_q", c_vp), ("run_tile", c_vp), ("run_static", c_vp), ("pm", c_vp),
                ("geo", c_vp),
                ("rec4", c_vp), ("d2", c_vp), ("pix", c_vp),
                ("gradr", c_vp), ("u", c_vp), ("u_out", c_vp), ("out", c_vp), ("out1", c_vp), ("rhs8", c_vp), ("rhs1", c_vp), ("tile_counter", c_vp),
                ("rec4_h", c_vp), ("d2_h", c_vp), ("pix_h", c_vp), ("e_split", c_ll), ("e_hbase", c_ll),
                ("jt_lanes", c_i), ("pad_", c_i)]


class SlmFwdArgs(C.Structure):
    _fields_ = [("xs", c_vp), ("G", c_ll), ("pair_gid", c_vp), ("pair_vm", c_vp), ("cams", c_vp), ("n_pairs", c_i),
                ("p", c_vp), ("sa", c_ll), ("sg", c_ll), ("pm", c_vp), ("gtab", c_vp),
                ("dsig", c_i), ("camf", c_vp)]


class SlmBackArgs(C.Structure):
    _fields_ = [("xs", c_vp), ("G", c_ll), ("gpo", c_vp), ("pair_vm", c_vp), ("cams", c_vp), ("pacc", c_vp), ("pacc1", c_vp),
                ("pair_run_off", c_vp), ("warp_g0", c_vp), ("pair_gid", c_vp), ("n_pairs", c_ll), ("gm", c_vp), ("gtab", c_vp),
                ("scale", c_f),
                ("p", c_vp), ("Mdiag", c_vp), ("lam", c_d), ("lam_out", c_i), ("out", c_vp), ("dot_part", c_vp),
                ("camf", c_vp)]


SPLAT_BYTES = 96
PAIR_GEO_BYTES = 32
PAIR_M_BYTES = 48
JT_D = 9          # J^T partials per run: 8 (32-byte records) + 1 (separate array)
DIAG_M = 40       # diag moment floats per run

# name -> (restype, argtypes)
_SIGS = {
    "slm_camera_size": (c_i, []), "slm_rastcfg_size": (c_i, []), "slm_splat_size": (c_i, []),
    "slm_pair_geo_size": (c_i, []), "slm_view_size": (c_i, []), "slm_raster_args_size": (c_i, []),
    "slm_resid_args_size": (c_i, []), "slm_tile_args_size": (c_i, []), "slm_back_args_size": (c_i, []),
    "slm_fwd_args_size": (c_i, []),
    "slm_diag_moment_floats": (c_i, []),
    "slm_preprocess": (c_i, [c_vp, c_ll, c_i, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "slm_sort_pairs_u64_workspace": (c_ll, [c_ll]),
    "slm_sort_pairs_u64": (c_i, [c_vp, c_ll, c_vp, c_vp, c_vp, c_vp, c_ll, c_i, c_i, c_vp]),
    "slm_tile_count": (c_i, [c_vp, c_vp, c_ll, c_vp, c_i, c_i, c_vp, c_vp]),
    "slm_tile_emit": (c_i, [c_vp, c_vp, c_ll, c_vp, c_i, c_i, c_vp, c_vp, c_vp]),
    "slm_tile_ranges": (c_i, [c_vp, c_ll, c_vp, c_i, c_vp]),
    "slm_raster_count": (c_i, [c_vp, c_vp]),
    "slm_raster_fill": (c_i, [c_vp, c_vp]),
    "slm_inst_count": (c_i, [c_vp, c_vp, c_ll, c_vp, c_vp, c_vp, c_vp]),
    "slm_runs_emit": (c_i, [c_vp, c_vp, c_vp, c_vp, c_vp, c_ll, c_ll, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "slm_tile_runs": (c_i, [c_vp, c_i, c_vp, c_vp, c_ll, c_i, c_vp, c_vp, c_vp, c_i, c_vp]),
    "slm_preprocess_views": (c_i, [c_vp, c_ll, c_i, c_vp, c_i, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "slm_tile_count_v": (c_i, [c_vp, c_ll, c_ll, c_vp, c_vp, c_vp, c_vp]),
    "slm_tile_emit_v": (c_i, [c_vp, c_vp, c_ll, c_ll, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "slm_sort_keys_u32_workspace": (c_ll, [c_ll]),
    "slm_sort_keys_u32": (c_i, [c_vp, c_ll, c_vp, c_vp, c_ll, c_i, c_i, c_vp]),
    "slm_residuals": (c_i, [c_vp, c_i, c_vp]),
    "slm_scan_i64_workspace": (c_ll, [c_ll]),
    "slm_scan_i64": (c_i, [c_vp, c_ll, c_vp, c_vp, c_ll, c_vp]),
    "slm_scan_i32_workspace": (c_ll, [c_ll]),
    "slm_scan_i32": (c_i, [c_vp, c_ll, c_vp, c_vp, c_ll, c_vp]),
    "slm_sort_pairs_u32_workspace": (c_ll, [c_ll]),
    "slm_sort_pairs_u32": (c_i, [c_vp, c_ll, c_vp, c_vp, c_vp, c_vp, c_ll, c_i, c_i, c_vp]),
    "slm_iota_u32": (c_i, [c_vp, c_ll, c_vp]),
    "slm_invert_perm": (c_i, [c_vp, c_ll, c_vp, c_vp]),
    "slm_pairs_prepare": (c_i, [c_vp, c_i, c_ll, c_vp, c_vp, c_vp, c_vp]),
    "slm_pairs_emit": (c_i, [c_vp, c_i, c_ll, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                             c_i, c_ll, c_vp]),
    "slm_export_view": (c_i, [c_vp, c_i, c_i, c_i, c_i, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i, c_i, c_vp,
                              c_vp, c_vp, c_ll, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "slm_apply_j": (c_i, [c_vp, c_vp]),
    "slm_apply_jt_runs": (c_i, [c_vp, c_vp]),
    "slm_jtwj_runs": (c_i, [c_vp, c_vp]),
    "slm_run_static": (c_i, [c_vp, c_ll, c_vp, c_vp, c_vp]),
    "slm_chunk_perm": (c_i, [c_vp, c_ll, c_vp, c_vp, c_vp, c_vp]),
    "slm_tile_chunks": (c_i, [c_vp, c_i, c_vp, c_vp, c_vp, c_vp, c_i, c_vp]),
    "slm_gauss_tab": (c_i, [c_vp, c_ll, c_i, c_vp, c_vp]),
    "slm_gauss_tab_floats": (c_i, [c_i]),
    "slm_diag_stream": (c_i, [c_vp, c_vp]),
    "slm_pair_forward": (c_i, [c_vp, c_i, c_vp]),
    "slm_backward_blocks": (c_i, [c_ll]),
    "slm_warp_bounds": (c_i, [c_vp, c_ll, c_i, c_vp, c_vp]),
    "slm_pair_backward": (c_i, [c_vp, c_i, c_i, c_vp]),
    "slm_vec_blocks": (c_i, []),
    "slm_gm_stride": (c_i, [c_i]),
    "slm_cameras_f32": (c_i, [c_vp, c_i, c_vp, c_vp]),
    "slm_gm_pack": (c_i, [c_vp, c_vp, c_ll, c_i, c_vp, c_i, c_vp]),
    "slm_pcg_pinit": (c_i, [c_vp, c_vp, c_vp, c_vp, c_ll, c_i, c_vp, c_i, c_vp]),
    "slm_pcg_pupdate": (c_i, [c_vp, c_vp, c_vp, c_vp, c_vp, c_ll, c_i, c_vp, c_i, c_vp]),
    "slm_pcg_update": (c_i, [c_i, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_d, c_vp, c_vp, c_i, c_vp, c_ll, c_vp]),
    "slm_pcg_finalize": (c_i, [c_i, c_vp, c_vp, c_vp]),
    "slm_combine_acc": (c_i, [c_vp, c_vp, c_vp, c_vp, c_ll, c_vp]),
    "slm_combine_fin": (c_i, [c_vp, c_vp, c_vp, c_ll, c_vp]),
    "slm_transpose_f32": (c_i, [c_vp, c_vp, c_ll, c_ll, c_vp]),
    "slm_transpose_f64": (c_i, [c_vp, c_vp, c_ll, c_ll, c_vp]),
    "slm_f64_to_f32": (c_i, [c_vp, c_vp, c_ll, c_vp]),
    "slm_axpy_scene": (c_i, [c_vp, c_vp, c_d, c_vp, c_ll, c_vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None
# count of kernel-launching entry points called (evidence for bench's gpu_launches)
launch_counter = {"calls": 0}


def load():
    """Load the shared library (CPU hosts can load it; no kernel runs without a GPU)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise SplatLMError(f"{LIB_PATH} missing: run `python -m paper_2409_12892_b200.build` "
                           "(there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_LOCAL)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    checks = {"slm_camera_size": SlmCamera, "slm_rastcfg_size": SlmRastCfg, "slm_view_size": SlmView,
              "slm_raster_args_size": SlmRasterArgs, "slm_resid_args_size": SlmResidArgs,
              "slm_tile_args_size": SlmTileArgs, "slm_back_args_size": SlmBackArgs, "slm_fwd_args_size": SlmFwdArgs}
    for fn, st in checks.items():
        if getattr(lib, fn)() != C.sizeof(st):
            raise SplatLMError(f"ABI mismatch: {fn} = {getattr(lib, fn)()} vs ctypes {C.sizeof(st)}")
    if lib.slm_splat_size() != SPLAT_BYTES or lib.slm_pair_geo_size() != PAIR_GEO_BYTES:
        raise SplatLMError("ABI mismatch in SlmSplat / SlmPairGeo")
    _lib = lib
    return lib


_STATUS = {1: ValueError, 2: RuntimeError, 3: LayoutError, 4: CacheOrderError, 5: ImageSizeError}


def check(status: int, what: str = ""):
    if status != 0:
        exc = _STATUS.get(status, RuntimeError)
        raise exc(f"libsplatlm_b200 {what} failed with status {status}")


def call(name: str, *args):
    """Invoke an entry point and raise on a non-zero status."""
    lib = load()
    launch_counter["calls"] += 1
    st = getattr(lib, name)(*args)
    check(st, name)
    return st


def ptr(t: torch.Tensor | None):
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


def off(t: torch.Tensor, elems: int):
    """Pointer to element `elems` of a contiguous tensor."""
    return C.c_void_p(t.data_ptr() + int(elems) * t.element_size())


def stream_ptr():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def byref(s):
    return C.byref(s)


def struct_tensor(arr, device) -> torch.Tensor:
    """Copy a ctypes array of structs to a device byte tensor."""
    raw = bytes(C.string_at(C.addressof(arr), C.sizeof(arr)))
    return torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(device)
