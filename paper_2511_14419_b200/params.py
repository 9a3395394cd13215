"""Parameter structs and error taxonomy of the RoI-extraction stage.

Python mirror of the reference's parameter structs, field for field, with the same
``validate()`` rules and the same error classes:

* ``DenoiseParams``  — /root/reference/proj/include/flowroi/denoise.hpp:11-24
* ``FlowParams``     — flow.hpp:12-30
* ``RoiParams``      — roi.hpp:20-38
* ``ExtractParams``  — roi.hpp:263-268 (``max_shift`` default kDefaultMaxShift = 16,
  registration.hpp:20)
* ``UsageError`` / ``DataError`` — ``usage_error`` / ``data_error``, core.hpp:14-22

``ExtractParams.to_c()`` packs them into the C ABI struct ``froi_params`` (include/froi/froi.h).
This module does not load the CUDA library, so it is importable on CPU-only hosts.
"""
from __future__ import annotations

import ctypes
import dataclasses
from dataclasses import dataclass, field

__all__ = [
    "UsageError", "DataError", "InternalError", "DenoiseParams", "FlowParams", "RoiParams",
    "ExtractParams", "Shift", "ExtractInfo", "StageTimes", "CParams", "CShift", "CFrameStats",
    "CStageTimes", "CKernelTimes", "GRADIENT_IMAGE", "GRADIENT_FLOW", "SHIFT_CONFIDENCE_THRESHOLD",
    "DEFAULT_MAX_SHIFT",
]

GRADIENT_IMAGE = 0  # SaliencyGradient::image (roi.hpp:18)
GRADIENT_FLOW = 1  # SaliencyGradient::flow
SHIFT_CONFIDENCE_THRESHOLD = 1.5  # kShiftConfidenceThreshold (registration.hpp:19)
DEFAULT_MAX_SHIFT = 16  # kDefaultMaxShift (registration.hpp:20)


class UsageError(ValueError):
    """flowroi::usage_error (core.hpp:14-17): bad parameters; CLI exit code 1."""


class DataError(ValueError):
    """flowroi::data_error (core.hpp:19-22): bad input data / shapes; CLI exit code 2."""


class InternalError(RuntimeError):
    """Anything else (CUDA failures included); CLI exit code 3."""


@dataclass
class DenoiseParams:
    enabled: bool = True
    median_radius: int = 1
    bilateral_sigma_spatial: float = 2.0
    bilateral_sigma_range: float = 0.04
    bilateral_radius: int = 2

    def validate(self) -> None:  # denoise.hpp:18-23
        if self.median_radius < 1 or self.bilateral_radius < 1:
            raise UsageError("denoise: radii must be >= 1")
        if self.bilateral_sigma_spatial <= 0 or self.bilateral_sigma_range <= 0:
            raise UsageError("denoise: sigmas must be > 0")


@dataclass
class FlowParams:
    pyramid_levels: int = 3
    pyramid_scale: float = 0.5
    window_size: int = 15
    iterations: int = 3
    poly_n: int = 5
    poly_sigma: float = 1.1

    def validate(self) -> None:  # flow.hpp:20-29
        if self.pyramid_levels < 1:
            raise UsageError("flow: pyramid_levels must be >= 1")
        if not (0.0 < self.pyramid_scale < 1.0):
            raise UsageError("flow: pyramid_scale must be in (0,1)")
        if self.window_size < 3 or self.window_size % 2 == 0:
            raise UsageError("flow: window_size must be odd and >= 3")
        if self.poly_n < 3 or self.poly_n % 2 == 0:
            raise UsageError("flow: poly_n must be odd and >= 3")
        if self.iterations < 1:
            raise UsageError("flow: iterations must be >= 1")
        if self.poly_sigma <= 0.0:
            raise UsageError("flow: poly_sigma must be > 0")


@dataclass
class RoiParams:
    roi_threshold: float = 0.2
    flow_weight: float = 0.7
    adjacent_factor: int = 0
    min_area: int = 20
    open_radius: int = 1
    close_radius: int = 1
    gradient_source: int = GRADIENT_IMAGE

    def validate(self) -> None:  # roi.hpp:29-37
        if not (0.0 < self.roi_threshold < 1.0):
            raise UsageError("roi: roi_threshold must be in (0,1)")
        if self.flow_weight < 0.0 or self.flow_weight > 1.0:
            raise UsageError("roi: flow_weight must be in [0,1]")
        if self.adjacent_factor < 0:
            raise UsageError("roi: adjacent_factor must be >= 0")
        if self.min_area < 0:
            raise UsageError("roi: min_area must be >= 0")
        if self.open_radius < 0 or self.close_radius < 0:
            raise UsageError("roi: radii must be >= 0")


class CParams(ctypes.Structure):
    """``froi_params`` (include/froi/froi.h)."""

    _fields_ = [
        ("denoise_enabled", ctypes.c_int),
        ("median_radius", ctypes.c_int),
        ("bilateral_sigma_spatial", ctypes.c_double),
        ("bilateral_sigma_range", ctypes.c_double),
        ("bilateral_radius", ctypes.c_int),
        ("pyramid_levels", ctypes.c_int),
        ("pyramid_scale", ctypes.c_double),
        ("window_size", ctypes.c_int),
        ("iterations", ctypes.c_int),
        ("poly_n", ctypes.c_int),
        ("poly_sigma", ctypes.c_double),
        ("roi_threshold", ctypes.c_double),
        ("flow_weight", ctypes.c_double),
        ("adjacent_factor", ctypes.c_int),
        ("min_area", ctypes.c_int),
        ("open_radius", ctypes.c_int),
        ("close_radius", ctypes.c_int),
        ("gradient_source", ctypes.c_int),
        ("max_shift", ctypes.c_int),
    ]


class CShift(ctypes.Structure):
    _fields_ = [("dx", ctypes.c_int), ("dy", ctypes.c_int), ("confidence", ctypes.c_double)]


class CFrameStats(ctypes.Structure):
    _fields_ = [
        ("dx", ctypes.c_int), ("dy", ctypes.c_int), ("confidence", ctypes.c_double),
        ("raw_fraction", ctypes.c_double), ("mask_count", ctypes.c_uint32),
        ("components", ctypes.c_uint32),
    ]


class CStageTimes(ctypes.Structure):
    _fields_ = [("denoise_ns", ctypes.c_uint64), ("flow_ns", ctypes.c_uint64),
                ("roi_ns", ctypes.c_uint64), ("encode_ns", ctypes.c_uint64)]


class CKernelTimes(ctypes.Structure):
    """``froi_kernel_times`` (include/froi/froi.h)."""
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "denoise_ns", "fft_forward_ns", "expand_ns", "register_ns", "expand_shifted_ns",
        "flow_iter_ns", "mask_ns", "pairs", "frames", "flow_iter_launches", "batches")]

    def as_dict(self) -> dict:
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


@dataclass
class ExtractParams:
    denoise: DenoiseParams = field(default_factory=DenoiseParams)
    flow: FlowParams = field(default_factory=FlowParams)
    roi: RoiParams = field(default_factory=RoiParams)
    max_shift: int = DEFAULT_MAX_SHIFT

    def validate(self) -> None:
        # extract_roi validates roi then flow (roi.hpp:312-313); denoise() validates its own.
        self.roi.validate()
        self.flow.validate()
        self.denoise.validate()

    def copy(self) -> "ExtractParams":
        return dataclasses.replace(self, denoise=dataclasses.replace(self.denoise),
                                   flow=dataclasses.replace(self.flow),
                                   roi=dataclasses.replace(self.roi))

    def to_c(self) -> CParams:
        d, f, r = self.denoise, self.flow, self.roi
        return CParams(int(bool(d.enabled)), d.median_radius, d.bilateral_sigma_spatial,
                       d.bilateral_sigma_range, d.bilateral_radius, f.pyramid_levels,
                       f.pyramid_scale, f.window_size, f.iterations, f.poly_n, f.poly_sigma,
                       r.roi_threshold, r.flow_weight, r.adjacent_factor, r.min_area,
                       r.open_radius, r.close_radius, int(r.gradient_source), self.max_shift)


@dataclass
class Shift:  # registration.hpp:13-17
    dx: int = 0
    dy: int = 0
    confidence: float = 1.0


@dataclass
class ExtractInfo:  # roi.hpp:271-274 (+ per-frame counts the GPU gathers for free)
    shifts: list = field(default_factory=list)
    raw_fractions: list = field(default_factory=list)
    mask_counts: list = field(default_factory=list)
    components: list = field(default_factory=list)


@dataclass
class StageTimes:  # roi.hpp:278-283, device time in ns
    denoise_ns: int = 0
    flow_ns: int = 0
    roi_ns: int = 0
    encode_ns: int = 0
