"""Bit-exact flow mode (froi_ctx_set_flow_exact, csrc/k_flow64.cu).

With it, compute_flow (flow.hpp:304-345) and extract_roi (roi.hpp:309-364) are byte-identical to
the reference: checked against the reference's own golden outputs (tests/golden, written by the
reference compiled in place) and against the oracle, which test_oracle_pin.py pins bit-exactly to
the reference.  Tolerance: none (np.array_equal on float32 flows and on masks).
"""
import os

import numpy as np
import pytest

from fixtures import cyclic_shift, textured_frame

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden_small.npz")


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


@pytest.fixture(scope="module")
def synth():
    from paper_2511_14419_b200 import synth as S
    return S


def _shift(f, dx, dy):
    h, w = f.shape
    return f[np.clip(np.arange(h) + dy, 0, h - 1)][:, np.clip(np.arange(w) + dx, 0, w - 1)]


def test_exact_flow_reference_golden(gpu, golden):
    u, v = gpu.compute_flow(golden["flow_a"], golden["flow_b"], exact=True)
    assert np.array_equal(u, golden["flow_u"]) and np.array_equal(v, golden["flow_v"])


def test_exact_sequence_reference_golden(gpu, golden):
    from paper_2511_14419_b200.params import ExtractInfo
    info = ExtractInfo()
    masks = gpu.extract_roi(golden["seq_frames"].astype(np.uint8), info=info, exact_flow=True)
    assert np.array_equal(masks, golden["seq_masks"])
    assert [(s.dx, s.dy, s.confidence) for s in info.shifts] == \
        [(int(a), int(b), float(c)) for a, b, c in golden["seq_shifts"]]
    assert np.array_equal(np.array(info.raw_fractions), golden["seq_fracs"])


@pytest.mark.parametrize("w,h,dx,dy,seed", [(96, 80, 2, 1, 21), (128, 96, -3, 2, 5), (65, 47, 1, -1, 3),
                                            (40, 36, 0, 1, 8), (200, 120, 4, -2, 11)])
def test_exact_flow_matches_oracle(gpu, oracle, w, h, dx, dy, seed):
    f = textured_frame(w, h, 8, seed)
    g = cyclic_shift(f, dx, dy)
    gu, gv = gpu.compute_flow(f, g, exact=True)
    ou, ov = oracle.compute_flow(f, g, 8)
    assert np.array_equal(gu, ou) and np.array_equal(gv, ov)


def test_exact_flow_params_and_16bit(gpu, oracle):
    from paper_2511_14419_b200.params import ExtractParams, FlowParams
    f = textured_frame(96, 88, 16, 4) >> 4  # 12-bit values in a depth-16 frame
    g = cyclic_shift(f, 2, -1)
    for levels, poly_n, poly_sigma, window, iters in [(1, 5, 1.1, 15, 3), (2, 7, 1.5, 9, 2),
                                                      (4, 5, 1.1, 5, 1), (3, 3, 0.8, 3, 4)]:
        p = FlowParams(pyramid_levels=levels, poly_n=poly_n, poly_sigma=poly_sigma,
                       window_size=window, iterations=iters)
        ep = ExtractParams()
        ep.flow = p
        gu, gv = gpu.compute_flow(f, g, p, depth=16, exact=True)
        ou, ov = oracle.compute_flow(f, g, 16, ep)
        assert np.array_equal(gu, ou) and np.array_equal(gv, ov), (levels, poly_n, window, iters)


def test_exact_flow_identical_frames_zero(gpu):
    f = textured_frame(64, 64, 8, 2)
    u, v = gpu.compute_flow(f, f, exact=True)
    assert not np.any(u) and not np.any(v)


def _exact_config(gpu, oracle, frames, depth, params, label):
    from paper_2511_14419_b200.params import ExtractInfo
    from oracle.oracle_py import extract_roi_job
    info = ExtractInfo()
    got = gpu.extract_roi(frames, params, info=info, depth=depth, exact_flow=True)
    want, shifts, fracs = extract_roi_job((frames, depth, params))
    assert [(s.dx, s.dy, s.confidence) for s in info.shifts] == \
        [(s.dx, s.dy, s.confidence) for s in shifts], label
    bad = [t for t in range(len(frames)) if not np.array_equal(got[t], want[t])]
    assert not bad, f"{label}: masks differ at frames {bad}"
    assert np.array_equal(np.array(info.raw_fractions), np.array(fracs)), label


def test_exact_extract_shifted_sequence(gpu, oracle):
    # registration shifts != 0: the shifted next frame's pyramid and expansions (pair slots)
    f = textured_frame(128, 96, 8, 12)
    frames = np.stack([cyclic_shift(f, 2 * t, -t) for t in range(4)])
    from paper_2511_14419_b200.params import ExtractParams
    _exact_config(gpu, oracle, frames, 8, ExtractParams(), "textured shifts")


def test_exact_c1_and_c2_prefix(gpu, oracle, synth):
    cfg = synth.config("C1")
    _exact_config(gpu, oracle, synth.well_frames(cfg, 0, 2), 8, cfg.params, "C1")
    cfg = synth.config("C2")
    _exact_config(gpu, oracle, synth.well_frames(cfg, 0, 4), 8, cfg.params, "C2[0:4]")


def test_exact_c4_pair_2048_16bit(gpu, oracle, synth):
    cfg = synth.config("C4")
    _exact_config(gpu, oracle, synth.well_frames(cfg, 0, 2), 16, cfg.params, "C4")


def test_exact_batches_and_lanes(gpu, oracle):
    """Multi-batch, two-lane exact runs equal the one-lane run and the oracle byte for byte."""
    from paper_2511_14419_b200.params import ExtractParams
    f = textured_frame(96, 96, 8, 7)
    frames = np.stack([cyclic_shift(f, t % 3, -(t % 2)) for t in range(9)])[None]
    want, _, _ = oracle.extract_roi(frames[0], 8, ExtractParams())
    outs = []
    for lanes in (1, 2):
        ctx = gpu.Context(96, 96, 8, ExtractParams(), max_pairs=2)
        try:
            ctx.set_lanes(lanes)
            ctx.set_flow_exact(True)
            assert ctx.flow_exact()
            m, _ = ctx.extract_wells(frames)
            outs.append(m[0])
            ctx.set_flow_exact(False)  # back to the fp32 flow on the same context
            m32, _ = ctx.extract_wells(frames)
            assert (m32[0] != want).mean() <= 1e-4
        finally:
            ctx.close()
    assert np.array_equal(outs[0], want) and np.array_equal(outs[1], want)


def test_exact_streaming_push(gpu, oracle):
    """Live acquisition (froi_stream_push) in the exact mode: pushes of 3, 1 and 2 frames give the
    oracle's masks for the whole sequence, frame-0 rule included."""
    from paper_2511_14419_b200 import _native
    from paper_2511_14419_b200.params import ExtractParams
    f = textured_frame(96, 96, 8, 8)
    frames = np.stack([cyclic_shift(f, t, -t) for t in range(6)]).astype(np.uint8)
    want, _, _ = oracle.extract_roi(frames, 8, ExtractParams())
    ctx = gpu.Context(96, 96, 8)
    try:
        ctx.set_flow_exact(True)
        _native.check(_native.lib.froi_stream_reset(ctx.handle, 1))
        got = []
        for chunk in (frames[0:3], frames[3:4], frames[4:6]):
            c = np.ascontiguousarray(chunk)
            out = np.empty((len(c), 96, 96), np.uint8)
            _native.check(_native.lib.froi_stream_push(ctx.handle, c.ctypes.data, 0, 1, 96 * 96, len(c),
                                                       0, out.ctypes.data, 0, None))
            got.append(out)
    finally:
        ctx.close()
    assert np.array_equal(np.concatenate(got), want)
