"""Host-side checks of the C ABI library (no GPU needed): it loads, exports every function the
header declares, validates parameters like the reference and reports geometry."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "froi", "froi.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(froi_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2511_14419_b200 import _native
    names = header_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(_native.lib, n), n
    assert set(names) == set(_native.exported_symbols())


def test_defaults_match_reference_structs():
    from paper_2511_14419_b200 import _native
    from paper_2511_14419_b200.params import CParams, ExtractParams
    c = CParams()
    _native.lib.froi_params_default(ctypes.byref(c))
    assert bytes(c) == bytes(ExtractParams().to_c())
    assert _native.lib.froi_params_validate(ctypes.byref(c)) == 0


@pytest.mark.parametrize("group,field,value", [
    ("roi", "roi_threshold", 0.0), ("roi", "roi_threshold", 1.0), ("roi", "flow_weight", 1.5),
    ("roi", "adjacent_factor", -1), ("roi", "min_area", -1), ("roi", "open_radius", -1),
    ("flow", "pyramid_levels", 0), ("flow", "pyramid_scale", 1.0), ("flow", "window_size", 14),
    ("flow", "poly_n", 4), ("flow", "iterations", 0), ("flow", "poly_sigma", 0.0),
    ("denoise", "median_radius", 0), ("denoise", "bilateral_sigma_range", 0.0),
])
def test_validation_matches_reference_rules(group, field, value):
    from paper_2511_14419_b200 import _native
    from paper_2511_14419_b200.params import ExtractParams, UsageError
    p = ExtractParams()
    setattr(getattr(p, group), field, value)
    with pytest.raises(UsageError):
        p.validate()
    c = p.to_c()
    assert _native.lib.froi_params_validate(ctypes.byref(c)) == 1
    with pytest.raises(UsageError):
        _native.check(1)


def test_pyramid_geometry():
    from paper_2511_14419_b200 import _native
    from paper_2511_14419_b200.params import ExtractParams

    def levels(w, h, n, scale=0.5):
        p = ExtractParams()
        p.flow.pyramid_levels = n
        p.flow.pyramid_scale = scale
        c = p.to_c()
        L = ctypes.c_int()
        ws = (ctypes.c_int * 16)()
        hs = (ctypes.c_int * 16)()
        assert _native.lib.froi_pyramid_levels(ctypes.byref(c), w, h, ctypes.byref(L), ws, hs) == 0
        return [(ws[i], hs[i]) for i in range(L.value)]

    assert levels(1024, 1024, 3) == [(1024, 1024), (512, 512), (256, 256)]
    assert levels(2048, 2048, 5)[-1] == (128, 128)
    assert levels(96, 96, 3) == [(96, 96), (48, 48)]  # stops before a level < 32 px
    assert levels(100, 70, 4, 0.7) == [(100, 70), (70, 49), (49, 34)]
    # 0.9 on 1024^2 would build 29 levels (build_pyramid, flow.hpp:289-298): the GPU tables hold
    # 16, so the geometry is refused with a usage error instead of silently capped
    p = ExtractParams()
    p.flow.pyramid_levels = 40
    p.flow.pyramid_scale = 0.9
    c = p.to_c()
    L = ctypes.c_int()
    assert _native.lib.froi_pyramid_levels(ctypes.byref(c), 1024, 1024, ctypes.byref(L), None, None) == 1
    assert b"16 levels" in _native.lib.froi_last_error()


def test_context_without_gpu_fails_cleanly():
    from paper_2511_14419_b200 import flowroi
    from paper_2511_14419_b200.params import InternalError
    if flowroi.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(InternalError):
        flowroi.Context(128, 128, 8)
