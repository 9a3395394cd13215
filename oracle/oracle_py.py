"""ctypes front-end of the CPU checkers (TEST INFRASTRUCTURE ONLY).

Two interchangeable backends with the same Python API:

* ``Oracle("port")``      — oracle/_build/libfroi_oracle.so, the C restatement
  (oracle/froi_oracle.c).  Always buildable (gcc only): ``ensure_built()`` runs ``make``.
* ``Oracle("reference")`` — oracle/_ref/libfroi_ref.so, the unmodified reference headers compiled
  in place (oracle/ref_shim.cpp).  Only buildable where /root/reference exists; the prebuilt
  .so travels with the repository snapshot to the GPU box.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may import this module.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

from paper_2511_14419_b200.params import (  # noqa: E402
    CParams, CShift, DataError, ExtractParams, InternalError, Shift, UsageError)

PORT_SO = os.path.join(_HERE, "_build", "libfroi_oracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libfroi_ref.so")

_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double


def ensure_built(reference: bool = False) -> None:
    """Build the restatement (and the in-place reference shim when the tree is present)."""
    target = "all" if reference else "oracle"
    if not os.path.exists(PORT_SO) or (reference and not os.path.exists(REF_SO)):
        subprocess.run(["make", "-s", "-C", _HERE, target], check=True)


def reference_available() -> bool:
    return os.path.exists(REF_SO)


def _ptr(a: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


def _check(status: int, what: str) -> None:
    if status == 0:
        return
    if status == 1:
        raise UsageError(what)
    if status == 2:
        raise DataError(what)
    raise InternalError(f"{what}: status {status}")


class Oracle:
    def __init__(self, kind: str = "port"):
        if kind not in ("port", "reference"):
            raise ValueError(kind)
        self.kind = kind
        if kind == "port":
            ensure_built(False)
            self.lib = ctypes.CDLL(PORT_SO)
            self.pre = "oracle_"
        else:
            if not os.path.exists(REF_SO):
                ensure_built(True)
            if not os.path.exists(REF_SO):
                raise FileNotFoundError(REF_SO)
            self.lib = ctypes.CDLL(REF_SO)
            self.pre = "ref_"
        self.lib_path = PORT_SO if kind == "port" else REF_SO

    def _fn(self, name, restype=ctypes.c_int):
        f = getattr(self.lib, self.pre + name)
        f.restype = restype
        return f

    # ---- denoise.hpp
    def denoise(self, frame: np.ndarray, depth: int, params: ExtractParams | None = None) -> np.ndarray:
        params = params or ExtractParams()
        f = np.ascontiguousarray(frame, dtype=np.uint16)
        out = np.empty_like(f)
        cp = params.to_c()
        h, w = f.shape
        _check(self._fn("denoise")(_ptr(f), _I(w), _I(h), _I(depth), ctypes.byref(cp), _ptr(out)),
               "denoise")
        return out

    # ---- registration.hpp
    def estimate_shift(self, ref: np.ndarray, mov: np.ndarray, depth: int = 8,
                       max_shift: int = 16) -> Shift:
        a = np.ascontiguousarray(ref, dtype=np.uint16)
        b = np.ascontiguousarray(mov, dtype=np.uint16)
        if a.shape != b.shape:
            raise DataError("estimate_shift: frames must share dimensions and depth")
        h, w = a.shape
        s = CShift()
        if self.kind == "port":
            st = self._fn("estimate_shift")(_ptr(a), _ptr(b), _I(w), _I(h), _I(max_shift),
                                           ctypes.byref(s))
        else:
            st = self._fn("estimate_shift")(_ptr(a), _ptr(b), _I(w), _I(h), _I(depth),
                                           _I(max_shift), ctypes.byref(s))
        _check(st, "estimate_shift")
        return Shift(s.dx, s.dy, s.confidence)

    # ---- flow.hpp
    def compute_flow(self, prev: np.ndarray, nxt: np.ndarray, depth: int,
                     params: ExtractParams | None = None):
        params = params or ExtractParams()
        a = np.ascontiguousarray(prev, dtype=np.uint16)
        b = np.ascontiguousarray(nxt, dtype=np.uint16)
        if a.shape != b.shape:
            raise DataError("compute_flow: frames must share dimensions")
        h, w = a.shape
        u = np.empty((h, w), np.float32)
        v = np.empty((h, w), np.float32)
        cp = params.to_c()
        _check(self._fn("compute_flow")(_ptr(a), _ptr(b), _I(w), _I(h), _I(depth),
                                        ctypes.byref(cp), _ptr(u), _ptr(v)), "compute_flow")
        return u, v

    def polynomial_expansion(self, img: np.ndarray, poly_n: int = 5, sigma: float = 1.1) -> np.ndarray:
        """Returns planes [6, h, w] in the order c, bx, by, a11, a12, a22."""
        im = np.ascontiguousarray(img, dtype=np.float64)
        h, w = im.shape
        planes = np.empty((6, h, w), np.float64)
        f = self._fn("polynomial_expansion", None if self.kind == "port" else ctypes.c_int)
        f(_ptr(im), _I(w), _I(h), _I(poly_n), _D(sigma), _ptr(planes))
        return planes

    # ---- roi.hpp
    def saliency(self, u, v, frame, depth: int, flow_weight: float = 0.7,
                 gradient_source: int = 0) -> np.ndarray:
        u = np.ascontiguousarray(u, dtype=np.float32)
        v = np.ascontiguousarray(v, dtype=np.float32)
        f = np.ascontiguousarray(frame, dtype=np.uint16)
        h, w = f.shape
        out = np.empty((h, w), np.float64)
        if self.kind == "port":
            st = self._fn("saliency")(_ptr(u), _ptr(v), _ptr(f), _I(w), _I(h), _I(depth),
                                      _D(flow_weight), _I(gradient_source), _ptr(out), None)
        else:
            st = self._fn("saliency")(_ptr(u), _ptr(v), _ptr(f), _I(w), _I(h), _I(depth),
                                      _D(flow_weight), _I(gradient_source), _ptr(out))
        _check(st, "saliency")
        return out

    def threshold_mask(self, sal: np.ndarray, t: float) -> np.ndarray:
        s = np.ascontiguousarray(sal, dtype=np.float64)
        h, w = s.shape
        m = np.empty((h, w), np.uint8)
        if self.kind == "port":
            st = self._fn("threshold_mask")(_ptr(s), _I(w), _I(h), _D(t), _ptr(m), None)
        else:
            st = self._fn("threshold_mask")(_ptr(s), _I(w), _I(h), _D(t), _ptr(m))
        _check(st, "threshold_mask")
        return m

    def morph_cleanup(self, mask: np.ndarray, open_radius=1, close_radius=1, min_area=20) -> np.ndarray:
        m = np.array(mask, dtype=np.uint8, copy=True, order="C")
        h, w = m.shape
        f = self._fn("morph_cleanup", None if self.kind == "port" else ctypes.c_int)
        f(_ptr(m), _I(w), _I(h), _I(open_radius), _I(close_radius), _I(min_area))
        return m

    # ---- dwt.hpp / codec.hpp (the codec side)
    def dwt_forward(self, frame: np.ndarray, depth: int, levels: int) -> np.ndarray:
        f = np.ascontiguousarray(frame, dtype=np.uint16)
        h, w = f.shape
        out = np.empty((h, w), np.int32)
        rc = self._fn("dwt_forward")(_ptr(f), _I(w), _I(h), _I(depth), _I(levels), _ptr(out))
        if rc == 1:
            raise UsageError("dwt: levels must be >= 1")
        if rc == 2:
            raise DataError("dwt: frame too small")
        if rc:
            raise RuntimeError("dwt_forward failed")
        return out

    def dwt_inverse(self, coeffs: np.ndarray, depth: int, levels: int) -> np.ndarray:
        c = np.ascontiguousarray(coeffs, dtype=np.int32)
        h, w = c.shape
        out = np.empty((h, w), np.uint16)
        if self._fn("dwt_inverse")(_ptr(c), _I(w), _I(h), _I(depth), _I(levels), _ptr(out)):
            raise RuntimeError("dwt_inverse failed")
        return out

    def map_mask_to_subbands(self, mask: np.ndarray, levels: int) -> list:
        m = np.ascontiguousarray(mask, dtype=np.uint8)
        h, w = m.shape
        dims, cw, ch = [], w, h
        for _ in range(levels):
            cw, ch = (cw + 1) // 2, (ch + 1) // 2
            dims.append((ch, cw))
        out = np.zeros(sum(a * b for a, b in dims), np.uint8)
        rt = ctypes.c_size_t if self.kind == "port" else ctypes.c_long
        n = self._fn("map_mask_to_subbands", rt)(_ptr(m), _I(w), _I(h), _I(levels), _ptr(out))
        if n != out.size:
            raise RuntimeError("map_mask_to_subbands failed")
        res, off = [], 0
        for a, b in dims:
            res.append(out[off:off + a * b].reshape(a, b).copy())
            off += a * b
        return res

    def component_areas(self, mask: np.ndarray) -> np.ndarray:
        m = np.ascontiguousarray(mask, dtype=np.uint8)
        h, w = m.shape
        if self.kind == "port":
            f = self._fn("label_components", ctypes.c_size_t)
            areas = np.zeros(w * h, np.uint64)
            n = f(_ptr(m), _I(w), _I(h), None, _ptr(areas), ctypes.c_size_t(w * h))
            return np.sort(areas[:n].astype(np.int64))
        f = self._fn("label_components", ctypes.c_long)
        areas = np.zeros(w * h, np.uint32)
        n = f(_ptr(m), _I(w), _I(h), _ptr(areas), ctypes.c_long(w * h))
        return np.sort(areas[:n].astype(np.int64))

    def mask_from_flow(self, u, v, raw, depth: int, dx: int, dy: int,
                       params: ExtractParams | None = None):
        """roi.hpp:337-345 for one pair (port only): returns (mask, debug dict)."""
        if self.kind != "port":
            raise NotImplementedError("mask_from_flow is a port-only tap")
        params = params or ExtractParams()
        u = np.ascontiguousarray(u, dtype=np.float32)
        v = np.ascontiguousarray(v, dtype=np.float32)
        f = np.ascontiguousarray(raw, dtype=np.uint16)
        h, w = f.shape
        m = np.empty((h, w), np.uint8)
        dbg = _PairDebug()
        cp = params.to_c()
        _check(self._fn("mask_from_flow")(_ptr(u), _ptr(v), _ptr(f), _I(w), _I(h), _I(depth),
                                          _I(dx), _I(dy), ctypes.byref(cp), _ptr(m),
                                          ctypes.byref(dbg)), "mask_from_flow")
        return m, dbg.as_dict()

    def extract_roi(self, frames: np.ndarray, depth: int, params: ExtractParams | None = None,
                    workers: int = 1):
        """Returns (masks [n,h,w] u8, shifts list[Shift], raw_fractions [n])."""
        params = params or ExtractParams()
        fr = np.ascontiguousarray(frames, dtype=np.uint16)
        n, h, w = fr.shape
        masks = np.empty((n, h, w), np.uint8)
        shifts = (CShift * n)()
        fracs = np.empty(n, np.float64)
        cp = params.to_c()
        if self.kind == "port":
            st = self._fn("extract_roi")(_ptr(fr), _I(n), _I(w), _I(h), _I(depth),
                                         ctypes.byref(cp), _I(workers), _ptr(masks), shifts,
                                         _ptr(fracs))
        else:
            st = self._fn("extract_roi")(_ptr(fr), _I(n), _I(w), _I(h), _I(depth),
                                         ctypes.byref(cp), _I(workers), _ptr(masks), shifts,
                                         _ptr(fracs), None)
        _check(st, "extract_roi")
        return masks, [Shift(s.dx, s.dy, s.confidence) for s in shifts], fracs

    # ---- reference-only helpers
    def generate_synthetic(self, n_cells=20, n_frames=50, width=512, height=512, depth=8,
                           speed=(1.0, 3.0), contrast=(20.0, 60.0), low_contrast_fraction=0.05,
                           temporal_noise_sigma=1.0, seed=7):
        """The reference's generate_synthetic (synthetic.hpp:135-290): frames, truth masks,
        track centres [cells, frames, 2] and radii."""
        if self.kind != "reference":
            raise NotImplementedError("generate_synthetic needs the reference build")
        frames = np.empty((n_frames, height, width), np.uint16)
        truth = np.empty((n_frames, height, width), np.uint8)
        xy = np.zeros((max(n_cells, 1), n_frames, 2), np.float64)
        radii = np.zeros(max(n_cells, 1), np.float64)
        f = self._fn("generate_synthetic")
        _check(f(_I(n_cells), _I(n_frames), _I(width), _I(height), _I(depth), _D(speed[0]),
                 _D(speed[1]), _D(contrast[0]), _D(contrast[1]), _D(low_contrast_fraction),
                 _D(temporal_noise_sigma), ctypes.c_uint64(seed), _ptr(frames), _ptr(truth),
                 _ptr(xy), _ptr(radii)), "generate_synthetic")
        return frames, truth, xy[:n_cells], radii[:n_cells]

    def hypot_restated(self, x: float, y: float) -> float:
        f = self._fn("hypot_restated", ctypes.c_double)
        return f(_D(x), _D(y))


class _ThresholdInfo(ctypes.Structure):
    _fields_ = [("target", ctypes.c_size_t), ("boundary", ctypes.c_double),
                ("count_greater", ctypes.c_size_t), ("count_equal", ctypes.c_size_t),
                ("ties_admitted", ctypes.c_size_t), ("degenerate", ctypes.c_int)]


class _PairDebug(ctypes.Structure):
    _fields_ = [("fmag_lo", ctypes.c_double), ("fmag_hi", ctypes.c_double),
                ("grad_lo", ctypes.c_double), ("grad_hi", ctypes.c_double),
                ("thr", _ThresholdInfo)]

    def as_dict(self):
        t = self.thr
        return dict(fmag_lo=self.fmag_lo, fmag_hi=self.fmag_hi, grad_lo=self.grad_lo,
                    grad_hi=self.grad_hi, target=t.target, boundary=t.boundary,
                    count_greater=t.count_greater, count_equal=t.count_equal,
                    ties_admitted=t.ties_admitted, degenerate=t.degenerate)


def extract_roi_job(args):
    """Process-pool helper (spawn-safe): (frames, depth, params[, workers]) -> extract_roi result."""
    frames, depth, params = args[:3]
    workers = args[3] if len(args) > 3 else (os.cpu_count() or 1)
    return Oracle("port").extract_roi(frames, depth, params, workers=workers)
