"""BASELINE configurations as seeded synthetic wells (BASELINE.json "configs").

``config(name)`` returns a ``SynthConfig`` for C1..C5; ``well_frames(cfg, well, n_frames)``
renders one well with the C generator in gen/synth.c (libfroi_synth.so, built by the same
Makefile as libfroi.so).  The ComplexEye recordings of the paper are not available; these seeded
scenes stand in for them with the shapes, sizes and value distributions BASELINE.json states.

Decisions recorded here: background noise is redrawn every frame; "flow
magnitude thresholds" map to ``roi_threshold`` and "dilation radii" to ``close_radius``; the
deeper pyramid of config 4 is ``pyramid_levels = 5``.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field, replace

import numpy as np

from .params import ExtractParams

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libfroi_synth.so")


class _Spec(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int), ("height", ctypes.c_int), ("sample_bytes", ctypes.c_int),
                ("data_max", ctypes.c_double), ("mu", ctypes.c_double), ("sigma", ctypes.c_double),
                ("n_cells", ctypes.c_int), ("cmean", ctypes.c_double), ("csd", ctypes.c_double),
                ("amin", ctypes.c_double), ("amax", ctypes.c_double), ("edge", ctypes.c_double),
                ("step", ctypes.c_double), ("persistence", ctypes.c_double),
                ("stationary_fraction", ctypes.c_double), ("flicker", ctypes.c_double),
                ("mode", ctypes.c_int), ("seed", ctypes.c_uint64)]


@dataclass
class SynthConfig:
    name: str
    width: int = 1024
    height: int = 1024
    depth: int = 8          # Frame::depth used for normalisation
    sample_bytes: int = 1
    data_max: float = 255.0
    mu: float = 100.0
    sigma: float = 5.0
    n_cells: int = 200
    cells_range: tuple | None = None  # per-well U{lo..hi} (config 3)
    cmean: float = 40.0
    csd: float = 10.0
    amin: float = 5.0
    amax: float = 12.0
    edge: float = 1.5
    step: float = 2.0
    persistence: float = 0.7
    stationary_fraction: float = 0.1
    flicker: float = 0.02
    mode: int = 0           # 0 walk, 1 single displacement, 2 zero motion
    seed: int = 1
    n_wells: int = 1
    n_frames: int = 2
    params: ExtractParams = field(default_factory=ExtractParams)

    def cells_for_well(self, well: int) -> int:
        if not self.cells_range:
            return self.n_cells
        lo, hi = self.cells_range
        z = (self.seed * 1_000_003 + well * 7919) & 0xFFFFFFFF
        return lo + z % (hi - lo + 1)


def config(name: str) -> SynthConfig:
    """BASELINE.json configs[0..4] as C1..C5 (C5 variants: C5-zero, C5-dense, C5-low)."""
    if name == "C1":
        return SynthConfig("C1", 512, 512, n_cells=60, mode=1, seed=1, n_frames=2,
                           stationary_fraction=0.0)
    if name == "C2":
        return SynthConfig("C2", n_cells=200, seed=2, n_frames=64)
    if name == "C3":
        return SynthConfig("C3", cells_range=(50, 400), seed=3000, n_wells=64, n_frames=450)
    if name == "C4":
        p = ExtractParams()
        p.flow.pyramid_levels = 5
        return SynthConfig("C4", 2048, 2048, depth=16, sample_bytes=2, data_max=4095.0, mu=1600.0,
                           sigma=80.0, n_cells=800, cmean=640.0, csd=160.0, step=6.0, seed=4000,
                           n_wells=16, n_frames=128, params=p)
    if name == "C5-zero":
        return SynthConfig("C5-zero", n_cells=200, mode=2, seed=5000, n_frames=2)
    if name == "C5-dense":
        return SynthConfig("C5-dense", n_cells=2000, mode=1, seed=5001, n_frames=2,
                           stationary_fraction=0.0)
    if name == "C5-low":
        return SynthConfig("C5-low", n_cells=200, cmean=8.0, csd=0.0, mode=1, seed=5002,
                           n_frames=2, stationary_fraction=0.0)
    raise KeyError(name)


def c5_grid() -> list:
    """C5 (iv): roi_threshold {0.1,0.2,0.3} x close_radius {1,2,3} x pyramid_levels {3,4}."""
    out = []
    for t in (0.1, 0.2, 0.3):
        for rc in (1, 2, 3):
            for L in (3, 4):
                p = ExtractParams()
                p.roi.roi_threshold = t
                p.roi.close_radius = rc
                p.flow.pyramid_levels = L
                out.append(((t, rc, L), p))
    return out


_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: build with make -C paper_2511_14419_b200/csrc")
        _lib = ctypes.CDLL(LIB_PATH)
        _lib.froi_synth_well.restype = ctypes.c_int
        _lib.froi_synth_well.argtypes = [ctypes.POINTER(_Spec), ctypes.c_int, ctypes.c_int,
                                         ctypes.c_void_p, ctypes.c_int]
        _lib.froi_fnv1a64.restype = ctypes.c_uint64
        _lib.froi_fnv1a64.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64]
    return _lib


def well_frames(cfg: SynthConfig, well: int = 0, n_frames: int | None = None,
                threads: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
    """Renders frames [n, H, W] (uint8 or uint16) of one well."""
    n = n_frames or cfg.n_frames
    dt = np.uint8 if cfg.sample_bytes == 1 else np.uint16
    if out is None:
        out = np.empty((n, cfg.height, cfg.width), dt)
    assert out.dtype == dt and out.shape == (n, cfg.height, cfg.width) and out.flags.c_contiguous
    s = _Spec(cfg.width, cfg.height, cfg.sample_bytes, cfg.data_max, cfg.mu, cfg.sigma,
              cfg.cells_for_well(well), cfg.cmean, cfg.csd, cfg.amin, cfg.amax, cfg.edge, cfg.step,
              cfg.persistence, cfg.stationary_fraction, cfg.flicker, cfg.mode, cfg.seed)
    th = threads or min(os.cpu_count() or 1, 64)
    if _load().froi_synth_well(ctypes.byref(s), well, n, out.ctypes.data, th) != 0:
        raise ValueError("bad synthetic spec")
    return out


def fnv1a64(a: np.ndarray, h: int = 0xCBF29CE484222325) -> int:
    """Content hash of the inputs (fnv1a64, core.hpp:155-162), recorded by the bench."""
    lib = _load()
    b = np.ascontiguousarray(a)
    return int(lib.froi_fnv1a64(b.ctypes.data, b.nbytes, ctypes.c_uint64(h)))


def scaled(cfg: SynthConfig, **kw) -> SynthConfig:
    return replace(cfg, **kw)
