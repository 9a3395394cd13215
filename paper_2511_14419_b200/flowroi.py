"""Host-side mirror of the reference's stage API (``namespace flowroi``), backed by the GPU.

Same names, argument meaning and error behaviour as the reference's inline C++ API, over numpy
arrays instead of ``Frame`` / ``RoiMask`` structs:

=========================================  ===============================================
reference (/root/reference/proj/include/)  here
=========================================  ===============================================
``extract_roi`` roi.hpp:309-364            ``extract_roi(seq, params, workers, info, timers)``
``compute_flow`` flow.hpp:304-345          ``compute_flow(prev, next, params, depth)``
``denoise`` denoise.hpp:84-90              ``denoise(frame, params, depth)``
``estimate_shift`` registration.hpp:46-97  ``estimate_shift(reference, moving, max_shift, depth)``
``polynomial_expansion`` flow.hpp:118-153  ``polynomial_expansion(img, poly_n, poly_sigma)``
``saliency`` roi.hpp:81-103                ``saliency(u, v, frame, flow_weight, source, depth)``
``threshold_mask`` roi.hpp:109-138         ``threshold_mask(map, roi_threshold)``
``morph_cleanup`` roi.hpp:237-246          ``morph_cleanup(mask, open_r, close_r, min_area)``
``label_components`` roi.hpp:184-234       ``component_areas(mask)`` (areas only)
``temporal_ensemble`` roi.hpp:249-261      ``temporal_ensemble(masks, t, k)``
=========================================  ===============================================

A frame is a 2-D uint8/uint16 array; ``depth`` (8 or 16) is ``Frame::depth`` and defaults to 8
like ``Frame`` (core.hpp:29) whatever the array dtype; a sample above the depth's maxval raises
DataError instead of being reinterpreted.  Masks are uint8 0/1 arrays (``RoiMask`` layout).  Every
call computes on the GPU through libfroi.so; errors raise UsageError / DataError exactly where the
reference throws usage_error / data_error.
"""
from __future__ import annotations

import contextlib
import ctypes
import threading
from dataclasses import dataclass

import numpy as np

from . import _native
from .params import (CFrameStats, CParams, CShift, CStageTimes, DataError, ExtractInfo,
                     ExtractParams, FlowParams, Shift, StageTimes, UsageError)

__all__ = [
    "Sequence", "extract_roi", "extract_wells", "compute_flow", "denoise", "estimate_shift",
    "polynomial_expansion", "saliency", "threshold_mask", "morph_cleanup", "component_areas",
    "temporal_ensemble", "mask_from_flow", "Context", "device_count",
]


@dataclass
class Sequence:
    """``flowroi::Sequence`` (core.hpp:61-75): frames [n, h, w] sharing one geometry."""
    frames: np.ndarray
    depth: int = 8
    frame_interval_s: float = 8.0

    def __len__(self) -> int:
        return int(self.frames.shape[0])


def device_count() -> int:
    n = ctypes.c_int(0)
    _native.lib.froi_device_count(ctypes.byref(n))
    return n.value


def _default_depth(a: np.ndarray) -> int:
    """Frame::depth defaults to 8 (core.hpp:29); 16-bit data must say depth=16."""
    return 8


def _frames_array(frames: np.ndarray, depth: int) -> np.ndarray:
    a = np.asarray(frames)
    if a.dtype not in (np.uint8, np.uint16):
        if np.issubdtype(a.dtype, np.integer):
            a = a.astype(np.uint16)
        else:
            raise DataError("frames must be uint8 or uint16 samples")
    if depth == 8 and a.dtype == np.uint16:
        if a.size and int(a.max()) > 255:
            raise DataError("frame sample exceeds the 8-bit depth")
        a = a.astype(np.uint8)
    return np.ascontiguousarray(a)


class Context:
    """A per-GPU context (froi_ctx): device arenas for one frame geometry and parameter set."""

    def __init__(self, width: int, height: int, depth: int = 8,
                 params: ExtractParams | None = None, device: int = 0, max_pairs: int = 0):
        self.params = (params or ExtractParams()).copy()
        self.width, self.height, self.depth, self.device = width, height, depth, device
        self._cp = self.params.to_c()
        self._h = ctypes.c_void_p()
        _native.check(_native.lib.froi_ctx_create(device, ctypes.byref(self._cp), width, height,
                                                  depth, max_pairs, ctypes.byref(self._h)),
                      "froi_ctx_create")
        self.lock = threading.RLock()
        self.users = 0  # holders of this context from the module cache (see _context)

    def close(self) -> None:
        # never while another thread runs on this context: ctypes releases the GIL inside the
        # native call, so froi_ctx_destroy must wait for the context's lock
        with self.lock:
            if self._h:
                _native.lib.froi_ctx_destroy(self._h)
                self._h = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    def stage_times(self) -> StageTimes:
        t = CStageTimes()
        _native.check(_native.lib.froi_ctx_stage_times(self._h, ctypes.byref(t)))
        return StageTimes(t.denoise_ns, t.flow_ns, t.roi_ns, t.encode_ns)

    def kernel_times(self) -> dict:
        from .params import CKernelTimes
        t = CKernelTimes()
        _native.check(_native.lib.froi_ctx_kernel_times(self._h, ctypes.byref(t)))
        return t.as_dict()

    def set_lanes(self, lanes: int) -> None:
        """1 or 2 execution lanes (two overlap consecutive batches; outputs are identical)."""
        _native.check(_native.lib.froi_ctx_set_lanes(self._h, int(lanes)))

    def set_fork(self, fork: bool) -> None:
        """Intra-batch overlap of the expansions with the FFT / registration (default on)."""
        _native.check(_native.lib.froi_ctx_set_fork(self._h, 1 if fork else 0))

    def set_flow_exact(self, exact: bool) -> None:
        """Bit-exact fp64 flow (k_flow64.cu; flows and masks byte-identical to the reference's)
        instead of the default fp32 flow within the stated tolerance.  Allocates its double
        buffers on first use."""
        _native.check(_native.lib.froi_ctx_set_flow_exact(self._h, 1 if exact else 0), "set_flow_exact")

    def flow_exact(self) -> bool:
        v = ctypes.c_int(0)
        _native.check(_native.lib.froi_ctx_get_flow_exact(self._h, ctypes.byref(v)))
        return bool(v.value)

    def stream(self) -> int:
        s = ctypes.c_void_p()
        _native.check(_native.lib.froi_ctx_stream(self._h, ctypes.byref(s)))
        return s.value or 0

    def extract_wells_device(self, d_frames: int, n_wells: int, n_frames: int, d_masks_pbm: int,
                             stats=None) -> None:
        """Device-resident variant (froi_extract_wells_device): pointers are device addresses."""
        with self.lock:
            _native.check(_native.lib.froi_extract_wells_device(
                self._h, ctypes.c_void_p(d_frames), 1 if self.depth == 8 else 2,
                self.width * self.height * (1 if self.depth == 8 else 2), n_wells, n_frames,
                ctypes.c_void_p(d_masks_pbm), stats), "extract_wells_device")

    def extract_wells_into(self, frames: np.ndarray, out: np.ndarray, stats=None, pbm: bool = True) -> None:
        """Host frames [wells, n, h, w] -> preallocated host masks (PBM rows by default)."""
        nw, n, h, w = frames.shape
        with self.lock:
            _native.check(_native.lib.froi_extract_wells(
                self._h, frames.ctypes.data, frames.itemsize, h * w * frames.itemsize, nw, n,
                1 if pbm else 0, out.ctypes.data, stats), "extract_roi")

    def launch_count(self) -> int:
        n = ctypes.c_uint64(0)
        _native.check(_native.lib.froi_ctx_launch_count(self._h, ctypes.byref(n)))
        return n.value

    def extract_wells(self, frames: np.ndarray, layout: str = "bytes"):
        """frames [wells, n, h, w] -> (masks, stats).  masks: [wells, n, h, w] bytes, or
        [wells, n, h, ceil(w/8)] PBM rows when layout == "pbm"."""
        a = _frames_array(frames, self.depth)
        if a.ndim == 3:
            a = a[None]
        nw, n, h, w = a.shape
        if (h, w) != (self.height, self.width):
            raise DataError("extract_roi: frame dimensions do not match the context")
        pbm = layout == "pbm"
        out = np.empty((nw, n, h, (w + 7) // 8 if pbm else w), np.uint8)
        stats = (CFrameStats * (nw * n))()
        with self.lock:
            _native.check(_native.lib.froi_extract_wells(
                self._h, a.ctypes.data, a.itemsize, h * w * a.itemsize, nw, n, 1 if pbm else 0,
                out.ctypes.data, stats), "extract_roi")
        return out, stats


_ctx_cache: dict = {}
_ctx_lock = threading.Lock()
_CTX_CACHE_MAX = 8


@contextlib.contextmanager
def _context(width: int, height: int, depth: int, params: ExtractParams, device: int = 0,
             exact_flow: bool = False):
    """A cached context, held for the duration of the ``with`` block: pinned against eviction
    (``users``) and locked, so concurrent callers of one context serialise and a context is only
    ever closed while nobody holds it.  ``exact_flow`` selects the bit-exact fp64 flow."""
    cp = params.to_c()
    key = (device, width, height, depth, bytes(cp), bool(exact_flow))
    with _ctx_lock:
        ctx = _ctx_cache.get(key)
        if ctx is None:
            idle = [k for k, c in _ctx_cache.items() if c.users == 0]
            while len(_ctx_cache) >= _CTX_CACHE_MAX and idle:
                _ctx_cache.pop(idle.pop(0)).close()
            ctx = Context(width, height, depth, params, device)
            if exact_flow:
                ctx.set_flow_exact(True)
            _ctx_cache[key] = ctx
        ctx.users += 1
    try:
        with ctx.lock:
            yield ctx
    finally:
        with _ctx_lock:
            ctx.users -= 1


def _split_shifts(stats, n: int) -> list:
    return [Shift(stats[i].dx, stats[i].dy, stats[i].confidence) for i in range(n)]


def extract_roi(seq, params: ExtractParams | None = None, workers: int = 1,
                info: ExtractInfo | None = None, timers: StageTimes | None = None,
                depth: int | None = None, exact_flow: bool = False) -> np.ndarray:
    """``flowroi::extract_roi`` (roi.hpp:309-364) on the GPU.  Returns masks [n, h, w] (uint8 0/1).

    ``workers`` keeps the reference signature; the output never depends on it
    (parallel.hpp:17-19).  A single sequence runs on one GPU.  ``exact_flow``: the bit-exact
    fp64 flow, so the masks are byte-identical to the reference's (slower)."""
    params = params or ExtractParams()
    params.roi.validate()
    params.flow.validate()
    if isinstance(seq, Sequence):
        frames, depth = seq.frames, seq.depth
    else:
        frames = np.asarray(seq)
        depth = depth or _default_depth(frames)
    if frames.ndim != 3:
        raise DataError("extract_roi: expected frames [n, h, w]")
    n, h, w = frames.shape
    if n < 2:
        raise DataError("extract_roi: sequence needs at least 2 frames")
    params.denoise.validate()
    with _context(w, h, depth, params, exact_flow=exact_flow) as ctx:
        masks, stats = ctx.extract_wells(frames[None])
        st = ctx.stage_times() if timers is not None else None
    if info is not None:
        info.shifts = _split_shifts(stats, n)
        info.raw_fractions = [stats[i].raw_fraction for i in range(n)]
        info.mask_counts = [stats[i].mask_count for i in range(n)]
        info.components = [stats[i].components for i in range(n)]
    if timers is not None:
        timers.denoise_ns += st.denoise_ns
        timers.flow_ns += st.flow_ns
        timers.roi_ns += st.roi_ns
    return masks[0]


def shard_wells(n_wells: int, devices: list[int]) -> dict:
    """Well w -> device devices[w mod len(devices)]; wells stay whole."""
    return {d: [w for w in range(n_wells) if w % len(devices) == k] for k, d in enumerate(devices)}


def extract_wells(frames: np.ndarray, params: ExtractParams | None = None, depth: int | None = None,
                  devices: list[int] | None = None, layout: str = "bytes", exact_flow: bool = False):
    """Independent wells [wells, n, h, w], sharded well-wise over ``devices`` (one host thread
    per GPU, no collective).  Returns (masks, list of per-well ExtractInfo)."""
    params = params or ExtractParams()
    params.validate()
    frames = np.asarray(frames)
    depth = depth or _default_depth(frames)
    nw, n, h, w = frames.shape
    devices = devices or [0]
    results: dict = {}
    errors: list = []

    def work(dev: int, wells: list[int]):
        try:
            with _context(w, h, depth, params, dev, exact_flow) as ctx:
                m, st = ctx.extract_wells(frames[wells], layout)
            results[dev] = (wells, m, st)
        except Exception as e:  # first error re-raised like parallel_for (parallel.hpp:31-48)
            errors.append(e)

    shards = shard_wells(nw, devices)
    threads = [threading.Thread(target=work, args=(d, ws)) for d, ws in shards.items() if ws]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    out = np.empty((nw, n, h, (w + 7) // 8 if layout == "pbm" else w), np.uint8)
    infos = [None] * nw
    for wells, m, st in results.values():
        for k, wi in enumerate(wells):
            out[wi] = m[k]
            s = st[k * n:(k + 1) * n]
            infos[wi] = ExtractInfo(shifts=[Shift(x.dx, x.dy, x.confidence) for x in s],
                                    raw_fractions=[x.raw_fraction for x in s],
                                    mask_counts=[x.mask_count for x in s],
                                    components=[x.components for x in s])
    return out, infos


def _u16(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=np.uint16)


def denoise(frame: np.ndarray, params: ExtractParams | None = None, depth: int | None = None) -> np.ndarray:
    """``flowroi::denoise`` (denoise.hpp:84-90)."""
    params = params or ExtractParams()
    params.denoise.validate()
    f = np.asarray(frame)
    depth = depth or _default_depth(f)
    h, w = f.shape
    a = _u16(f)
    out = np.empty_like(a)
    with _small_ctx(w, h, depth, params.copy()) as ctx:
        _native.check(_native.lib.froi_denoise(ctx.handle, a.ctypes.data, out.ctypes.data), "denoise")
    return out.astype(f.dtype) if f.dtype == np.uint8 else out


def estimate_shift(reference: np.ndarray, moving: np.ndarray, max_shift: int = 16,
                   depth: int | None = None) -> Shift:
    """``flowroi::estimate_shift`` (registration.hpp:46-97)."""
    a, b = np.asarray(reference), np.asarray(moving)
    if a.shape != b.shape:
        raise DataError("estimate_shift: frames must share dimensions and depth")
    h, w = a.shape
    if max_shift < 1 or max_shift >= min(w, h) // 4:
        raise UsageError("estimate_shift: max_shift must be in [1, min(w,h)/4)")
    depth = depth or _default_depth(a)
    p = ExtractParams()
    p.max_shift = max_shift
    s = CShift()
    a16, b16 = _u16(a), _u16(b)
    with _context(w, h, depth, p) as ctx:
        _native.check(_native.lib.froi_estimate_shift(ctx.handle, a16.ctypes.data, b16.ctypes.data,
                                                      max_shift, ctypes.byref(s)), "estimate_shift")
    return Shift(s.dx, s.dy, s.confidence)


def compute_flow(prev: np.ndarray, nxt: np.ndarray, params: FlowParams | ExtractParams | None = None,
                 depth: int | None = None, exact: bool = False):
    """``flowroi::compute_flow`` (flow.hpp:304-345): returns (u, v) float32 [h, w].  ``exact``:
    the bit-exact fp64 flow (identical to the reference's) instead of the fp32 one."""
    ep = ExtractParams()
    if isinstance(params, ExtractParams):
        ep = params.copy()
    elif isinstance(params, FlowParams):
        ep.flow = params
    ep.flow.validate()
    a, b = np.asarray(prev), np.asarray(nxt)
    if a.shape != b.shape:
        raise DataError("compute_flow: frames must share dimensions")
    h, w = a.shape
    depth = depth or _default_depth(a)
    ep.max_shift = max(1, min(ep.max_shift, min(w, h) // 4 - 1))
    u = np.empty((h, w), np.float32)
    v = np.empty((h, w), np.float32)
    a16, b16 = _u16(a), _u16(b)
    with _context(w, h, depth, ep, exact_flow=exact) as ctx:
        _native.check(_native.lib.froi_compute_flow(ctx.handle, a16.ctypes.data, b16.ctypes.data,
                                                    u.ctypes.data, v.ctypes.data), "compute_flow")
    return u, v


def polynomial_expansion(img: np.ndarray, poly_n: int = 5, poly_sigma: float = 1.1) -> np.ndarray:
    """``flowroi::polynomial_expansion`` (flow.hpp:118-153) in fp32: planes [6, h, w] in the
    order c, bx, by, a11, a12, a22."""
    im = np.ascontiguousarray(img, dtype=np.float32)
    h, w = im.shape
    ep = ExtractParams()
    ep.flow.poly_n = poly_n
    ep.flow.poly_sigma = poly_sigma
    ep.flow.validate()
    ep.max_shift = max(1, min(ep.max_shift, min(w, h) // 4 - 1))
    planes = np.empty((6, h, w), np.float32)
    with _context(w, h, 8, ep) as ctx:
        _native.check(_native.lib.froi_polynomial_expansion(ctx.handle, im.ctypes.data,
                                                            planes.ctypes.data), "polynomial_expansion")
    return planes


def _small_ctx(w: int, h: int, depth: int, ep: ExtractParams) -> Context:
    ep.max_shift = max(1, min(ep.max_shift, min(w, h) // 4 - 1))
    return _context(w, h, depth, ep)


def saliency(u: np.ndarray, v: np.ndarray, frame: np.ndarray, flow_weight: float = 0.7,
             gradient_source: int = 0, depth: int | None = None) -> np.ndarray:
    """``flowroi::saliency`` (roi.hpp:81-103): float64 map."""
    f = np.asarray(frame)
    h, w = f.shape
    if np.shape(u) != (h, w) or np.shape(v) != (h, w):
        raise DataError("saliency: flow/frame dimension mismatch")
    depth = depth or _default_depth(f)
    ep = ExtractParams()
    ep.roi.flow_weight = flow_weight
    ep.roi.gradient_source = gradient_source
    ep.roi.validate()
    out = np.empty((h, w), np.float64)
    uu = np.ascontiguousarray(u, dtype=np.float32)
    vv = np.ascontiguousarray(v, dtype=np.float32)
    f16 = _u16(f)
    with _small_ctx(w, h, depth, ep) as ctx:
        _native.check(_native.lib.froi_saliency(ctx.handle, uu.ctypes.data, vv.ctypes.data,
                                                f16.ctypes.data, out.ctypes.data), "saliency")
    return out


def threshold_mask(sal: np.ndarray, roi_threshold: float) -> np.ndarray:
    """``flowroi::threshold_mask`` (roi.hpp:109-138)."""
    if not (0.0 < roi_threshold < 1.0):
        raise UsageError("threshold_mask: roi_threshold must be in (0,1)")
    m = np.ascontiguousarray(sal, dtype=np.float64)
    h, w = m.shape
    out = np.empty((h, w), np.uint8)
    with _small_ctx(w, h, 8, ExtractParams()) as ctx:
        _native.check(_native.lib.froi_threshold_mask(ctx.handle, m.ctypes.data, roi_threshold,
                                                      out.ctypes.data), "threshold_mask")
    return out


def morph_cleanup(mask: np.ndarray, open_radius: int = 1, close_radius: int = 1,
                  min_area: int = 20) -> np.ndarray:
    """``flowroi::morph_cleanup`` (roi.hpp:237-246)."""
    m = np.array(mask, dtype=np.uint8, copy=True, order="C")
    h, w = m.shape
    with _small_ctx(w, h, 8, ExtractParams()) as ctx:
        _native.check(_native.lib.froi_morph_cleanup(ctx.handle, m.ctypes.data, open_radius,
                                                     close_radius, min_area), "morph_cleanup")
    return m


def morph_open(mask: np.ndarray, radius: int) -> np.ndarray:
    """``flowroi::morph_open`` (roi.hpp:179)."""
    return morph_cleanup(mask, radius, 0, 0)


def morph_close(mask: np.ndarray, radius: int) -> np.ndarray:
    """``flowroi::morph_close`` (roi.hpp:180)."""
    return morph_cleanup(mask, 0, radius, 0)


def component_areas(mask: np.ndarray) -> np.ndarray:
    """Areas of the 8-connected components (``label_components``, roi.hpp:184-234), sorted."""
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    h, w = m.shape
    n = ctypes.c_size_t(0)
    areas = np.zeros(w * h, np.uint32)
    with _small_ctx(w, h, 8, ExtractParams()) as ctx:
        _native.check(_native.lib.froi_component_areas(ctx.handle, m.ctypes.data, areas.ctypes.data,
                                                       areas.size, ctypes.byref(n)), "component_areas")
    return np.sort(areas[:n.value].astype(np.int64))


def temporal_ensemble(masks: np.ndarray, t: int, k: int) -> np.ndarray:
    """``flowroi::temporal_ensemble`` (roi.hpp:249-261): union of masks [t-k, t+k]."""
    m = np.ascontiguousarray(masks, dtype=np.uint8)
    n, h, w = m.shape
    if t < 0 or t >= n:
        raise DataError("temporal_ensemble: index out of range")
    out = np.empty_like(m)
    with _small_ctx(w, h, 8, ExtractParams()) as ctx:
        _native.check(_native.lib.froi_temporal_ensemble(ctx.handle, m.ctypes.data, n, k,
                                                         out.ctypes.data), "temporal_ensemble")
    return out[t]


def mask_from_flow(u: np.ndarray, v: np.ndarray, raw: np.ndarray, dx: int = 0, dy: int = 0,
                   params: ExtractParams | None = None, depth: int | None = None):
    """Mask stage of one pair (roi.hpp:340-345) from a given flow: returns (mask, stats)."""
    params = params or ExtractParams()
    f = np.asarray(raw)
    h, w = f.shape
    depth = depth or _default_depth(f)
    ep = params.copy()
    mask = np.empty((h, w), np.uint8)
    st = CFrameStats()
    uu = np.ascontiguousarray(u, dtype=np.float32)
    vv = np.ascontiguousarray(v, dtype=np.float32)
    f16 = _u16(f)
    with _small_ctx(w, h, depth, ep) as ctx:
        _native.check(_native.lib.froi_mask_from_flow(ctx.handle, uu.ctypes.data, vv.ctypes.data,
                                                      f16.ctypes.data, dx, dy, mask.ctypes.data,
                                                      ctypes.byref(st)), "mask_from_flow")
    return mask, dict(mask_count=st.mask_count, components=st.components,
                      raw_fraction=st.raw_fraction)


# ---------------------------------------------------------------- wire formats and the report
def save_flo(path: str, u: np.ndarray, v: np.ndarray) -> None:
    """FLO1 flow dump (``save_flo``, flow.hpp:347-366): b"FLO1", u32 LE width and height, then
    row-major (u, v) pairs as f32 LE."""
    u32 = np.ascontiguousarray(u, dtype="<f4")
    v32 = np.ascontiguousarray(v, dtype="<f4")
    if u32.shape != v32.shape or u32.ndim != 2:
        raise DataError("save_flo: u and v must be 2-D arrays of one shape")
    h, w = u32.shape
    inter = np.empty((h, w, 2), "<f4")
    inter[..., 0] = u32
    inter[..., 1] = v32
    try:
        with open(path, "wb") as f:
            f.write(b"FLO1" + np.array([w, h], "<u4").tobytes() + inter.tobytes())
    except OSError as e:
        raise DataError(f"cannot write {path}: {e}") from e


def load_flo(path: str) -> tuple[np.ndarray, np.ndarray]:
    """Reads a FLO1 file (``load_flo``, flow.hpp:368-389) -> (u, v) float32 arrays."""
    try:
        data = open(path, "rb").read()
    except OSError as e:
        raise DataError(f"cannot open {path}") from e
    if data[:4] != b"FLO1":
        raise DataError(f"{path}: not a FLO1 file")
    if len(data) < 12:
        raise DataError(f"{path}: bad FLO1 header")
    w, h = (int(x) for x in np.frombuffer(data[4:12], "<u4"))
    if w <= 0 or h <= 0:
        raise DataError(f"{path}: bad FLO1 header")
    if len(data) < 12 + 8 * w * h:
        raise DataError(f"{path}: truncated FLO1 data")
    inter = np.frombuffer(data[12:12 + 8 * w * h], "<f4").reshape(h, w, 2)
    return inter[..., 0].copy(), inter[..., 1].copy()


def save_pbm(path: str, mask: np.ndarray, width: int | None = None) -> None:
    """P4 mask file (``save_pbm``, pgm.hpp:127-138): b"P4\\n<w> <h>\\n" + rows packed MSB first,
    padded to whole bytes.  `mask` is [h, w] 0/1 bytes, or [h, ceil(w/8)] PBM rows (the
    FROI_MASK_PBM layout the GPU writes) together with `width`."""
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    if width is None:
        h, w = m.shape
        rows = np.packbits(m != 0, axis=1)
    else:
        h, w = m.shape[0], int(width)
        if m.shape[1] != (w + 7) // 8:
            raise DataError("save_pbm: PBM rows do not match the width")
        rows = m
    try:
        with open(path, "wb") as f:
            f.write(f"P4\n{w} {h}\n".encode() + rows.tobytes())
    except OSError as e:
        raise DataError(f"cannot write {path}: {e}") from e


def extract_report_frames(masks: np.ndarray, info: ExtractInfo) -> list[dict]:
    """The per-frame rows of the extract-roi report (tools/flowroi.cpp:186-196): mask fraction,
    8-connected component count of the final mask (``label_components``, on the GPU) and the
    registration shift."""
    m = np.asarray(masks)
    rows = []
    for i in range(m.shape[0]):
        s = info.shifts[i]
        rows.append({"index": i, "mask_fraction": float((m[i] != 0).mean()),
                     "components": int(component_areas(m[i]).size),
                     "shift": {"dx": int(s.dx), "dy": int(s.dy), "confidence": float(s.confidence)}})
    return rows


# ---------------------------------------------------------------- codec side
def dwt_forward(frame: np.ndarray, levels: int = 5, depth: int | None = None) -> np.ndarray:
    """Reversible 5/3 DWT on the GPU (``dwt_forward``, dwt.hpp:113-141): DC-shifted int32
    coefficients in the canonical in-place layout (coarser levels in the top-left quadrant)."""
    f = _u16(frame)
    d = depth or _default_depth(np.asarray(frame))
    h, w = f.shape
    out = np.empty((h, w), np.int32)
    with _small_ctx(w, h, d, ExtractParams()) as ctx:
        _native.check(_native.lib.froi_dwt_forward(ctx.handle, f.ctypes.data, int(levels), out.ctypes.data),
                      "dwt_forward")
    return out


def dwt_inverse(coeffs: np.ndarray, levels: int = 5, depth: int = 8) -> np.ndarray:
    """Inverse of ``dwt_forward`` (``dwt_inverse``, dwt.hpp:143-171) -> uint16 frame."""
    c = np.ascontiguousarray(coeffs, dtype=np.int32)
    h, w = c.shape
    out = np.empty((h, w), np.uint16)
    with _small_ctx(w, h, depth, ExtractParams()) as ctx:
        _native.check(_native.lib.froi_dwt_inverse(ctx.handle, c.ctypes.data, int(levels), out.ctypes.data),
                      "dwt_inverse")
    return out


def map_mask_to_subbands(mask: np.ndarray, levels: int = 5) -> list[np.ndarray]:
    """RoI coefficient masks per level (``map_mask_to_subbands``, codec.hpp:152-171), level 1
    (finest) first: 2x2 OR down-sampling then a radius-2 square dilation, on the GPU."""
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    h, w = m.shape
    dims, cw, ch = [], w, h
    for _ in range(int(levels)):
        cw, ch = (cw + 1) // 2, (ch + 1) // 2
        dims.append((ch, cw))
    out = np.zeros(sum(a * b for a, b in dims), np.uint8)
    n = ctypes.c_size_t(0)
    with _small_ctx(w, h, 8, ExtractParams()) as ctx:
        _native.check(_native.lib.froi_map_mask_to_subbands(ctx.handle, m.ctypes.data, int(levels),
                                                            out.ctypes.data, out.size, ctypes.byref(n)),
                      "map_mask_to_subbands")
    res, off = [], 0
    for a, b in dims:
        res.append(out[off:off + a * b].reshape(a, b).copy())
        off += a * b
    return res
