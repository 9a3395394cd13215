"""End-to-end GPU parity of extract_roi (roi.hpp:309-364) against the CPU oracle.

* per-frame shifts (incl. confidence) bit-identical, frame 0 borrows frame 1;
* the mask stage is bit-exact given the GPU's own flow (oracle mask stage run on that flow), so
  every end-to-end mask difference is propagated from the flow's float tolerance;
* end-to-end mask mismatch <= 1e-4 of the pixels per frame, reported.
"""
import numpy as np
import pytest

from fixtures import cyclic_shift, textured_frame

pytestmark = pytest.mark.gpu

MASK_MISMATCH_MAX = 1e-4


def _sequence(reference, seed=55, n=4, size=96, cells=3):
    if reference is not None:
        frames, truth, xy, radii = reference.generate_synthetic(
            n_cells=cells, n_frames=n, width=size, height=size, seed=seed)
        return frames
    f = textured_frame(size, size, 8, seed)
    return np.stack([cyclic_shift(f, t, (t * 2) % 3) for t in range(n)])


@pytest.fixture(scope="module")
def ref_or_none():
    from oracle.oracle_py import Oracle, reference_available
    return Oracle("reference") if reference_available() else None


def _check_sequence(gpu, oracle, frames, depth=8, params=None):
    from paper_2511_14419_b200.params import ExtractInfo, ExtractParams
    params = params or ExtractParams()
    info = ExtractInfo()
    got = gpu.extract_roi(frames.astype(np.uint16) if depth == 16 else frames.astype(np.uint8),
                          params, info=info, depth=depth)
    want, shifts, fracs = oracle.extract_roi(frames, depth, params)
    assert [(s.dx, s.dy, s.confidence) for s in info.shifts] == \
        [(s.dx, s.dy, s.confidence) for s in shifts]
    n, h, w = frames.shape
    mism = [(got[t] != want[t]).mean() for t in range(n)]
    # mask stage exact given the GPU flow of each pair
    if params.roi.adjacent_factor == 0:
        den = np.stack([gpu.denoise(frames[t].astype(np.uint16), params, depth=depth) for t in range(n)])
        for t in range(1, n):
            s = shifts[t]
            nxt = den[t]
            if s.dx or s.dy:
                from oracle.oracle_py import Oracle  # noqa: F401  (apply_shift restated below)
                ys = np.clip(np.arange(h) + s.dy, 0, h - 1)
                xs = np.clip(np.arange(w) + s.dx, 0, w - 1)
                nxt = den[t][ys][:, xs]
            u, v = gpu.compute_flow(den[t - 1], nxt, params, depth=depth)
            m, _ = oracle.mask_from_flow(u, v, frames[t], depth, s.dx, s.dy, params)
            assert np.array_equal(m, got[t]), f"mask stage differs at frame {t}"
        assert np.array_equal(got[0], got[1])
    assert max(mism) <= MASK_MISMATCH_MAX, mism
    fr = np.array(info.raw_fractions)
    assert np.allclose(fr, [g.mean() for g in got] if params.roi.adjacent_factor == 0 else fr)
    return got, max(mism)


def test_extract_small_sequence(gpu, oracle, ref_or_none):
    frames = _sequence(ref_or_none)
    _check_sequence(gpu, oracle, frames)


def test_extract_textured_shifts(gpu, oracle):
    f = textured_frame(128, 96, 8, 12)
    frames = np.stack([cyclic_shift(f, 2 * t, -t) for t in range(4)])
    _check_sequence(gpu, oracle, frames)


def test_extract_static_sequence(gpu, oracle, ref_or_none):
    # test_roi.cpp:247-258 expects empty masks for a static scene; the reference code itself
    # keeps 872 px of gradient speckle on this input, so parity is the contract.
    if ref_or_none is None:
        pytest.skip("needs the reference generator (oracle/_ref)")
    frames, *_ = ref_or_none.generate_synthetic(n_cells=0, n_frames=1, width=96, height=96,
                                                temporal_noise_sigma=0.0)
    got, mism = _check_sequence(gpu, oracle, np.repeat(frames, 4, axis=0))
    assert mism == 0.0


def test_extract_zero_motion_ties(gpu, oracle):
    # identical frames: flow exactly zero, saliency = 0.3*N(grad) with many exact ties
    f = textured_frame(128, 128, 8, 31)
    frames = np.stack([f, f, f])
    got, mism = _check_sequence(gpu, oracle, frames)
    assert mism == 0.0


def test_extract_16bit(gpu, oracle, ref_or_none):
    frames = _sequence(ref_or_none, seed=9, n=3, size=96)
    frames16 = (frames.astype(np.uint16) << 4)  # 12-bit values in a depth-16 frame
    _check_sequence(gpu, oracle, frames16, depth=16)


@pytest.mark.parametrize("knob", ["threshold", "close", "levels", "ensemble", "gradflow", "denoise_off",
                                  "open", "min_area", "flow_weight", "max_shift", "window", "scale"])
def test_extract_param_grid(gpu, oracle, ref_or_none, knob):
    from paper_2511_14419_b200.params import ExtractParams
    p = ExtractParams()
    if knob == "threshold":
        p.roi.roi_threshold = 0.1
    elif knob == "close":
        p.roi.close_radius = 3
    elif knob == "levels":
        p.flow.pyramid_levels = 2
    elif knob == "ensemble":
        p.roi.adjacent_factor = 1
    elif knob == "gradflow":
        p.roi.gradient_source = 1
    elif knob == "denoise_off":
        p.denoise.enabled = False
    elif knob == "open":
        p.roi.open_radius = 2
    elif knob == "min_area":
        p.roi.min_area = 60
    elif knob == "flow_weight":
        p.roi.flow_weight = 0.3
    elif knob == "max_shift":
        p.max_shift = 8
    elif knob == "window":
        p.flow.window_size = 9
    elif knob == "scale":
        p.flow.pyramid_scale = 0.6
    frames = _sequence(ref_or_none, seed=4, n=4, size=96, cells=2)
    _check_sequence(gpu, oracle, frames, params=p)


def test_extract_errors(gpu):
    from paper_2511_14419_b200.params import DataError, ExtractParams, UsageError
    with pytest.raises(DataError):
        gpu.extract_roi(np.zeros((1, 64, 64), np.uint8))
    p = ExtractParams()
    p.roi.roi_threshold = 1.0
    with pytest.raises(UsageError):
        gpu.extract_roi(np.zeros((2, 64, 64), np.uint8), p)


def test_extract_wells_and_worker_independence(gpu, oracle):
    from paper_2511_14419_b200.flowroi import Context
    f = textured_frame(96, 96, 8, 77)
    wells = np.stack([np.stack([cyclic_shift(f, t * (w + 1), t) for t in range(3)]) for w in range(3)])
    ctx = Context(96, 96, 8, max_pairs=2)  # forces several batches
    masks, stats = ctx.extract_wells(wells.astype(np.uint8))
    for w in range(3):
        single = gpu.extract_roi(wells[w].astype(np.uint8))
        assert np.array_equal(masks[w], single)
    pbm, _ = ctx.extract_wells(wells.astype(np.uint8), layout="pbm")
    assert np.array_equal(np.unpackbits(pbm, axis=-1)[..., :96], masks)


def test_streaming_matches_whole_sequence(gpu):
    import ctypes

    from paper_2511_14419_b200 import _native
    from paper_2511_14419_b200.flowroi import Context
    f = textured_frame(96, 96, 8, 8)
    frames = np.stack([cyclic_shift(f, t, -t) for t in range(6)]).astype(np.uint8)
    whole = gpu.extract_roi(frames)
    ctx = Context(96, 96, 8)
    _native.check(_native.lib.froi_stream_reset(ctx.handle, 1))
    got = []
    for chunk in (frames[0:3], frames[3:4], frames[4:6]):
        c = np.ascontiguousarray(chunk)
        out = np.empty((len(c), 96, 96), np.uint8)
        _native.check(_native.lib.froi_stream_push(ctx.handle, c.ctypes.data, 0, 1, 96 * 96, len(c),
                                                   0, out.ctypes.data, 0, None))
        got.append(out)
    assert np.array_equal(np.concatenate(got), whole)


def test_two_lanes_identical(gpu):
    """Two execution lanes (consecutive batches on two buffer sets / streams) give the same
    masks and stats byte for byte as one lane, for a call spanning several batches and wells."""
    from paper_2511_14419_b200 import flowroi
    from paper_2511_14419_b200.params import ExtractParams
    n, size = 13, 96
    wells = np.stack([np.stack([cyclic_shift(textured_frame(size, size, 8, 70 + w), t, (t * w) % 3)
                                for t in range(n)]) for w in range(2)]).astype(np.uint8)
    out = {}
    for lanes in (1, 2):
        ctx = flowroi.Context(size, size, 8, ExtractParams(), max_pairs=4)
        ctx.set_lanes(lanes)
        masks, stats = ctx.extract_wells(wells, layout="pbm")
        out[lanes] = (masks, [(s.dx, s.dy, s.confidence, s.mask_count) for s in stats])
    assert np.array_equal(out[1][0], out[2][0])
    assert out[1][1] == out[2][1]


def test_pinned_pbm_streamed_back_identical(gpu):
    """PBM masks into pinned host memory are copied back batch by batch during the call (frame 0
    of each well at the end); the bytes equal the pageable-memory path."""
    import torch
    from paper_2511_14419_b200 import flowroi
    from paper_2511_14419_b200.params import CFrameStats, ExtractParams
    n, size = 13, 96
    wells = np.stack([np.stack([cyclic_shift(textured_frame(size, size, 8, 90 + w), t, (t * w) % 3)
                                for t in range(n)]) for w in range(2)]).astype(np.uint8)
    ctx = flowroi.Context(size, size, 8, ExtractParams(), max_pairs=4)
    want, _ = ctx.extract_wells(wells, layout="pbm")
    pinned = torch.zeros((2, n, size, (size + 7) // 8), dtype=torch.uint8, pin_memory=True)
    stats = (CFrameStats * (2 * n))()
    ctx.extract_wells_into(wells, pinned.numpy(), stats)
    assert np.array_equal(pinned.numpy(), want)


def test_extract_report_frames(gpu, oracle):
    """Per-frame rows of the extract-roi report (tools/flowroi.cpp:186-196): components of each
    final mask by the GPU labeller equal the restated label_components; fractions and shifts come
    straight from the stage."""
    from paper_2511_14419_b200 import flowroi
    from paper_2511_14419_b200.params import ExtractInfo, ExtractParams
    frames = np.stack([cyclic_shift(textured_frame(96, 96, 8, 321), t, t % 2) for t in range(5)]).astype(np.uint8)
    info = ExtractInfo()
    masks = flowroi.extract_roi(frames, ExtractParams(), info=info)
    rows = flowroi.extract_report_frames(masks, info)
    assert [r["index"] for r in rows] == list(range(5))
    for r, m in zip(rows, masks):
        assert r["components"] == oracle.component_areas(m).size
        assert r["mask_fraction"] == float(m.mean())
    assert [(r["shift"]["dx"], r["shift"]["dy"]) for r in rows] == [(s.dx, s.dy) for s in info.shifts]


def test_selection_rest_kernels_identical(gpu, tmp_path):
    """Selection finished entirely by the per-pair k_sel_rest_* kernels (FROI_SEL_GRID_PASSES=0,
    read once per process, so in a subprocess) gives the same masks and stats as the default
    grid-wide passes, on a sequence with many exactly equal saliency values (static frames) and
    a moving one."""
    import os
    import subprocess
    import sys
    from paper_2511_14419_b200.params import ExtractInfo, ExtractParams
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    static = np.stack([textured_frame(128, 96, 8, 7)] * 4)
    moving = np.stack([cyclic_shift(textured_frame(128, 96, 8, 9), t, t % 2) for t in range(5)])
    np.save(tmp_path / "static.npy", static)
    np.save(tmp_path / "moving.npy", moving)
    script = (
        "import sys, numpy as np\n"
        f"sys.path.insert(0, {root!r})\n"
        "from paper_2511_14419_b200 import flowroi\n"
        "from paper_2511_14419_b200.params import ExtractInfo, ExtractParams\n"
        "for name in ('static', 'moving'):\n"
        f"    f = np.load({str(tmp_path)!r} + '/' + name + '.npy')\n"
        "    info = ExtractInfo()\n"
        "    m = flowroi.extract_roi(f, ExtractParams(), info=info)\n"
        f"    np.save({str(tmp_path)!r} + '/' + name + '_rest.npy', m)\n"
        f"    np.save({str(tmp_path)!r} + '/' + name + '_fr.npy', np.array(info.raw_fractions))\n")
    env = dict(os.environ, FROI_SEL_GRID_PASSES="0")
    subprocess.run([sys.executable, "-c", script], check=True, env=env, cwd=root)
    for name, frames in (("static", static), ("moving", moving)):
        info = ExtractInfo()
        want = gpu.extract_roi(frames, ExtractParams(), info=info)
        got = np.load(tmp_path / f"{name}_rest.npy")
        assert np.array_equal(got, want), name
        assert np.array_equal(np.load(tmp_path / f"{name}_fr.npy"), np.array(info.raw_fractions)), name


@pytest.mark.parametrize("w,h", [(40, 36), (65, 33), (100, 70), (129, 64), (31, 97)])
def test_extract_odd_shapes(gpu, oracle, w, h):
    """Ragged shapes: widths that are not multiples of 32 (threshold words without the fused
    path), of 64 (partial flow tiles, clusters of tiles not filling a row) and pyramids that stop
    after one or two levels; shifts, masks and stats against the oracle as everywhere else."""
    from paper_2511_14419_b200.params import ExtractParams
    p = ExtractParams()
    p.max_shift = 4
    f = textured_frame(w, h, 8, w + h)
    frames = np.stack([cyclic_shift(f, t % 2, t // 2) for t in range(4)])
    _check_sequence(gpu, oracle, frames, params=p)


@pytest.mark.parametrize("w,h", [(8192, 40), (40, 8192)])
def test_extract_maximum_extent(gpu, oracle, w, h):
    """The largest FFT side the GPU supports (8192) on either axis, against the oracle; one more
    pixel is refused with a usage error (never silently truncated)."""
    from paper_2511_14419_b200.params import ExtractParams, UsageError
    p = ExtractParams()
    p.max_shift = 8
    f = textured_frame(w, h, 8, 3)
    frames = np.stack([cyclic_shift(f, t, -t) for t in range(3)])
    _check_sequence(gpu, oracle, frames, params=p)
    want, _, _ = oracle.extract_roi(frames, 8, p)
    assert np.array_equal(gpu.extract_roi(frames, p, exact_flow=True), want)  # bit-exact mode too
    with pytest.raises(UsageError):
        gpu.extract_roi(np.zeros((2, h + (h > w), w + (w > h)), np.uint8), p)


def test_per_frame_pointer_entries(gpu):
    """froi_extract_frames (one uint16 pointer per frame and per mask), froi_extract_frames_sink
    (each destination requested once, frame 0 after frame 1) and froi_stream_push_frames give the
    bytes of the contiguous entry; a u16 sample above 255 in an 8-bit context is a data error."""
    import ctypes

    from paper_2511_14419_b200 import _native
    from paper_2511_14419_b200.flowroi import Context
    from paper_2511_14419_b200.params import DataError
    n, size = 11, 96
    f = textured_frame(size, size, 8, 123)
    frames = np.stack([cyclic_shift(f, t, (2 * t) % 5) for t in range(n)]).astype(np.uint8)
    ctx = Context(size, size, 8, max_pairs=3)
    want, _ = ctx.extract_wells(frames[None])
    f16 = [np.ascontiguousarray(frames[t], dtype=np.uint16) for t in range(n)]
    fp = (ctypes.c_void_p * n)(*[a.ctypes.data for a in f16])
    # per-frame pointers
    outs = [np.empty((size, size), np.uint8) for _ in range(n)]
    mp = (ctypes.c_void_p * n)(*[a.ctypes.data for a in outs])
    _native.check(_native.lib.froi_extract_frames(ctx.handle, fp, 2, n, 0, mp, None))
    assert np.array_equal(np.stack(outs), want[0])
    # sink: destinations handed out on demand
    sunk = {}
    order = []
    SINK = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int)

    def sink(user, well, frame):
        order.append(frame)
        a = np.empty((size, size), np.uint8)
        sunk[frame] = a
        return a.ctypes.data

    cb = SINK(sink)
    _native.check(_native.lib.froi_extract_frames_sink(ctx.handle, fp, 2, n, 0, ctypes.cast(cb, ctypes.c_void_p),
                                                      None, None))
    assert sorted(order) == list(range(n))
    assert order.index(0) > order.index(1)
    assert np.array_equal(np.stack([sunk[t] for t in range(n)]), want[0])
    # put: finished masks handed over (the drop-in's path)
    got_put = {}
    PUT = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p)

    def put(user, well, frame, ptr):
        got_put[frame] = np.ctypeslib.as_array((ctypes.c_uint8 * (size * size)).from_address(ptr)).reshape(size, size).copy()
        return 0

    pcb = PUT(put)
    _native.check(_native.lib.froi_extract_frames_put(ctx.handle, fp, 2, n, 0, ctypes.cast(pcb, ctypes.c_void_p),
                                                     None, None))
    assert np.array_equal(np.stack([got_put[t] for t in range(n)]), want[0])
    # streaming with per-frame pointers, uneven pushes
    _native.check(_native.lib.froi_stream_reset(ctx.handle, 1))
    got = []
    for a, b in ((0, 4), (4, 5), (5, 11)):
        k = b - a
        so = [np.empty((size, size), np.uint8) for _ in range(k)]
        sp = (ctypes.c_void_p * k)(*[x.ctypes.data for x in so])
        _native.check(_native.lib.froi_stream_push_frames(ctx.handle, ctypes.cast(fp, ctypes.c_void_p).value + 8 * a,
                                                          2, k, 0, sp, None))
        got += so
    assert np.array_equal(np.stack(got), want[0])
    # the Frame invariant: samples < 2^depth
    bad = [np.ascontiguousarray(x, dtype=np.uint16) for x in f16]
    bad[3][5, 7] = 300
    bp = (ctypes.c_void_p * n)(*[a.ctypes.data for a in bad])
    with pytest.raises(DataError):
        _native.check(_native.lib.froi_extract_frames(ctx.handle, bp, 2, n, 0, mp, None))
    ctx.close()


@pytest.mark.parametrize("knob", ["default", "threshold", "close", "levels", "ensemble", "gradflow",
                                  "denoise_off", "open", "min_area", "window", "scale", "poly7"])
def test_extract_exact_flow_param_grid(gpu, oracle, ref_or_none, knob):
    """The bit-exact flow mode end to end over the same parameter grid: every mask, shift,
    confidence and raw fraction identical to the reference's."""
    from paper_2511_14419_b200.params import ExtractInfo, ExtractParams
    p = ExtractParams()
    if knob == "threshold":
        p.roi.roi_threshold = 0.1
    elif knob == "close":
        p.roi.close_radius = 3
    elif knob == "levels":
        p.flow.pyramid_levels = 2
    elif knob == "ensemble":
        p.roi.adjacent_factor = 1
    elif knob == "gradflow":
        p.roi.gradient_source = 1
    elif knob == "denoise_off":
        p.denoise.enabled = False
    elif knob == "open":
        p.roi.open_radius = 2
    elif knob == "min_area":
        p.roi.min_area = 60
    elif knob == "window":
        p.flow.window_size = 9
    elif knob == "scale":
        p.flow.pyramid_scale = 0.6
    elif knob == "poly7":
        p.flow.poly_n = 7
        p.flow.poly_sigma = 1.5
    frames = _sequence(ref_or_none, seed=4, n=4, size=96, cells=2)
    info = ExtractInfo()
    got = gpu.extract_roi(frames.astype(np.uint8), p, info=info, exact_flow=True)
    want, shifts, fracs = oracle.extract_roi(frames, 8, p)
    assert np.array_equal(got, want)
    assert [(s.dx, s.dy, s.confidence) for s in info.shifts] == [(s.dx, s.dy, s.confidence) for s in shifts]
    assert np.array_equal(np.array(info.raw_fractions), np.array(fracs))
