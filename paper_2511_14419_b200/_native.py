"""ctypes binding of libfroi.so (the C ABI declared in include/froi/froi.h).

The library is built in-tree by ``make -C paper_2511_14419_b200/csrc`` (or
``__graft_entry__.build()``).  There is no fallback: if the shared library is missing this
module raises ImportError, and every compute entry fails with InternalError when no CUDA device
is usable.
"""
from __future__ import annotations

import ctypes
import os

from .params import (CFrameStats, CKernelTimes, CParams, CShift, CStageTimes, DataError,
                     InternalError, UsageError)

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libfroi.so")
# profiling A/B only (profiles/tools/stage_ab.py): another in-tree build of the same library
LIB_PATH = os.environ.get("FROI_LIB", LIB_PATH)

_P = ctypes.c_void_p
_I = ctypes.c_int
_SZ = ctypes.c_size_t

# name -> (restype, argtypes); mirrors include/froi/froi.h
SIGNATURES = {
    "froi_version": (ctypes.c_char_p, []),
    "froi_last_error": (ctypes.c_char_p, []),
    "froi_params_default": (None, [ctypes.POINTER(CParams)]),
    "froi_params_validate": (_I, [ctypes.POINTER(CParams)]),
    "froi_pyramid_levels": (_I, [ctypes.POINTER(CParams), _I, _I, ctypes.POINTER(_I), _P, _P]),
    "froi_device_count": (_I, [ctypes.POINTER(_I)]),
    "froi_ctx_create": (_I, [_I, ctypes.POINTER(CParams), _I, _I, _I, _I, ctypes.POINTER(_P)]),
    "froi_ctx_destroy": (None, [_P]),
    "froi_ctx_get_params": (_I, [_P, ctypes.POINTER(CParams)]),
    "froi_ctx_set_params": (_I, [_P, ctypes.POINTER(CParams)]),
    "froi_ctx_stage_times": (_I, [_P, ctypes.POINTER(CStageTimes)]),
    "froi_ctx_launch_count": (_I, [_P, ctypes.POINTER(ctypes.c_uint64)]),
    "froi_ctx_kernel_times": (_I, [_P, ctypes.POINTER(CKernelTimes)]),
    "froi_ctx_stream": (_I, [_P, ctypes.POINTER(_P)]),
    "froi_ctx_set_lanes": (_I, [_P, ctypes.c_int]),
    "froi_ctx_set_fork": (_I, [_P, ctypes.c_int]),
    "froi_ctx_set_flow_exact": (_I, [_P, ctypes.c_int]),
    "froi_ctx_get_flow_exact": (_I, [_P, ctypes.POINTER(ctypes.c_int)]),
    "froi_dwt_forward": (_I, [_P, _P, ctypes.c_int, _P]),
    "froi_dwt_inverse": (_I, [_P, _P, ctypes.c_int, _P]),
    "froi_dwt_forward_device": (_I, [_P, _P, ctypes.c_int, ctypes.c_int, _P]),
    "froi_map_mask_to_subbands": (_I, [_P, _P, ctypes.c_int, _P, ctypes.c_size_t,
                                       ctypes.POINTER(ctypes.c_size_t)]),
    "froi_extract_roi": (_I, [_P, _P, _I, _SZ, _I, _I, _P, _P]),
    "froi_extract_wells": (_I, [_P, _P, _I, _SZ, _I, _I, _I, _P, _P]),
    "froi_extract_wells_device": (_I, [_P, _P, _I, _SZ, _I, _I, _P, _P]),
    "froi_extract_frames": (_I, [_P, _P, _I, _I, _I, _P, _P]),
    "froi_extract_frames_sink": (_I, [_P, _P, _I, _I, _I, _P, _P, _P]),
    "froi_extract_frames_put": (_I, [_P, _P, _I, _I, _I, _P, _P, _P]),
    "froi_stream_reset": (_I, [_P, _I]),
    "froi_stream_push": (_I, [_P, _P, _I, _I, _SZ, _I, _I, _P, _I, _P]),
    "froi_stream_push_frames": (_I, [_P, _P, _I, _I, _I, _P, _P]),
    "froi_denoise": (_I, [_P, _P, _P]),
    "froi_estimate_shift": (_I, [_P, _P, _P, _I, ctypes.POINTER(CShift)]),
    "froi_compute_flow": (_I, [_P, _P, _P, _P, _P]),
    "froi_polynomial_expansion": (_I, [_P, _P, _P]),
    "froi_saliency": (_I, [_P, _P, _P, _P, _P]),
    "froi_threshold_mask": (_I, [_P, _P, ctypes.c_double, _P]),
    "froi_morph_cleanup": (_I, [_P, _P, _I, _I, _I]),
    "froi_component_areas": (_I, [_P, _P, _P, _SZ, ctypes.POINTER(_SZ)]),
    "froi_mask_from_flow": (_I, [_P, _P, _P, _P, _I, _I, _P, ctypes.POINTER(CFrameStats)]),
    "froi_debug_pair_stats": (_I, [_P, _I, _P, _I]),
    "froi_temporal_ensemble": (_I, [_P, _P, _I, _I, _P]),
}


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        if "FROI_LIB" in os.environ and not hasattr(lib, name):
            continue  # an older build under A/B comparison
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def last_error() -> str:
    msg = lib.froi_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = "") -> None:
    """Maps ABI status codes onto the reference's error taxonomy (core.hpp:14-22)."""
    if status == 0:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if status == 1:
        raise UsageError(msg)
    if status == 2:
        raise DataError(msg)
    raise InternalError(msg)


def exported_symbols() -> list[str]:
    return list(SIGNATURES)
