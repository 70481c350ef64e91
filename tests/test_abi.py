"""CPU: the C-ABI library loads, every symbol include/splatlm_b200.h declares
is exported, and the ctypes struct layouts match the C ones.  No kernel runs."""
import ctypes
import os
import re

import pytest

from paper_2409_12892_b200 import _lib

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "splatlm_b200.h")


def declared_symbols():
    text = open(HDR).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(slm_[a-z0-9_]+)\s*\(", text)))


def test_library_builds_and_loads():
    from paper_2409_12892_b200 import build
    build.build()
    lib = _lib.load()
    assert lib is not None


def test_every_declared_symbol_is_exported():
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) > 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the ctypes binding covers exactly the header
    assert set(_lib.EXPORTED) == set(syms)


def test_struct_layouts():
    lib = _lib.load()
    assert lib.slm_camera_size() == ctypes.sizeof(_lib.SlmCamera)
    assert lib.slm_raster_args_size() == ctypes.sizeof(_lib.SlmRasterArgs)
    assert lib.slm_resid_args_size() == ctypes.sizeof(_lib.SlmResidArgs)
    assert lib.slm_tile_args_size() == ctypes.sizeof(_lib.SlmTileArgs)
    assert lib.slm_back_args_size() == ctypes.sizeof(_lib.SlmBackArgs)
    assert lib.slm_splat_size() == 96 and lib.slm_pair_geo_size() == 32


def test_workspace_queries_do_not_crash_without_gpu():
    lib = _lib.load()
    assert lib.slm_scan_i64_workspace(1 << 20) >= 0
    assert lib.slm_sort_pairs_u32_workspace(1 << 20) >= 0


def test_error_mapping():
    from paper_2409_12892_b200.errors import CacheOrderError, ImageSizeError, LayoutError
    with pytest.raises(ValueError):
        _lib.check(1, "x")
    with pytest.raises(LayoutError):
        _lib.check(3, "x")
    with pytest.raises(CacheOrderError):
        _lib.check(4, "x")
    with pytest.raises(ImageSizeError):
        _lib.check(5, "x")
    with pytest.raises(RuntimeError):
        _lib.check(2, "x")
