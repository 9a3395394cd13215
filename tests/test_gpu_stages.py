"""GPU parity per stage: every sub-operator through the C ABI against the CPU oracle.

Contracts:
* denoise, registration (shift AND confidence), saliency, threshold, morphology, CCL areas and
  the whole mask stage given a flow: bit-exact;
* flow (fp32 on the GPU vs fp64 reference): max |du|,|dv| <= 2e-2 px and mean EPE <= 1e-3 px;
  identical frames give exactly zero flow.
"""
import numpy as np
import pytest

from fixtures import Rng, cyclic_shift, random_frame, random_mask, textured_frame

pytestmark = pytest.mark.gpu

FLOW_MAX_ABS = 2e-2
FLOW_MEAN_EPE = 1e-3


def _impulses(f, seed, count=40, value=255):
    g = f.copy()
    r = Rng(seed)
    h, w = g.shape
    for _ in range(count):
        g[r.next_below(h), r.next_below(w)] = value
    return g


# ---------------------------------------------------------------- denoise (denoise.hpp)
@pytest.mark.parametrize("w,h,depth,seed", [(96, 80, 8, 21), (33, 21, 8, 8), (130, 67, 16, 5),
                                             (64, 64, 16, 9)])
def test_denoise_bit_exact(gpu, oracle, w, h, depth, seed):
    f = textured_frame(w, h, depth, seed)
    if depth == 16:
        f = (f >> 4).astype(np.uint16)  # 12-bit data in a depth-16 frame (BASELINE config 4)
    for frame in (f, _impulses(f, seed, value=(1 << depth) - 1), random_frame(w, h, 8, seed)):
        got = gpu.denoise(frame.astype(np.uint16), depth=depth)
        want = oracle.denoise(frame, depth)
        assert np.array_equal(got, want)


def _c3_frames(n):
    from paper_2511_14419_b200 import synth
    return synth.well_frames(synth.config("C3"), 0, n)


def test_denoise_full_frame(gpu, oracle):
    """1024^2 u8 frames of the bench's workload and a uniform-noise frame: every pixel equal."""
    frames = _c3_frames(2)
    r = Rng(77)
    noisy = np.array([[r.next_below(256) for _ in range(256)] for _ in range(256)], np.uint8)
    for frame in (frames[0], frames[1], noisy):
        got = gpu.denoise(frame.astype(np.uint16), depth=8)
        want = oracle.denoise(frame, 8)
        assert np.array_equal(got, want)


@pytest.mark.parametrize("mr,br,ss,sr", [(2, 2, 2.0, 0.04), (1, 3, 1.5, 0.1), (3, 1, 3.0, 0.02),
                                          (1, 7, 4.0, 0.3), (2, 4, 0.7, 0.01), (1, 2, 2.0, 0.5)])
def test_denoise_params_bit_exact(gpu, oracle, mr, br, ss, sr):
    """Denoise off the defaults (the generic runtime-radius kernel, and the default-radius fast
    kernel under other sigmas): median radius 1-3, bilateral radius 1-7, spatial / range sigmas
    from 0.7 to 4 and 0.01 to 0.5 -- bit-exact on 8-bit, 12-bit-in-16 and impulse frames."""
    from paper_2511_14419_b200.params import ExtractParams
    p = ExtractParams()
    p.denoise.median_radius = mr
    p.denoise.bilateral_radius = br
    p.denoise.bilateral_sigma_spatial = ss
    p.denoise.bilateral_sigma_range = sr
    for depth, seed in ((8, 3), (16, 4)):
        f = textured_frame(77, 61, depth, seed)
        if depth == 16:
            f = (f >> 4).astype(np.uint16)
        for frame in (f, _impulses(f, seed, value=(1 << depth) - 1)):
            got = gpu.denoise(frame.astype(np.uint16), p, depth=depth)
            want = oracle.denoise(frame, depth, p)
            assert np.array_equal(got, want), (mr, br, ss, sr, depth)


def test_denoise_constant_identity(gpu):
    f = np.full((18, 24), 77, np.uint16)
    assert np.array_equal(gpu.denoise(f, depth=8), f)


def test_denoise_disabled_is_copy(gpu):
    from paper_2511_14419_b200.params import ExtractParams
    p = ExtractParams()
    p.denoise.enabled = False
    f = textured_frame(33, 21, 16, 8)
    assert np.array_equal(gpu.denoise(f, p, depth=16), f)


# ---------------------------------------------------------------- registration
def test_shift_identity_and_cyclic(gpu, oracle):
    f = textured_frame(96, 96, 8, 1)
    s = gpu.estimate_shift(f, f, 16)
    assert (s.dx, s.dy) == (0, 0) and s.confidence > 1.5
    assert s == oracle.estimate_shift(f, f, 8, 16)
    f = textured_frame(128, 128, 8, 2)
    g = cyclic_shift(f, 3, -2)
    s = gpu.estimate_shift(f, g, 16)
    assert (s.dx, s.dy) == (3, -2)
    assert s == oracle.estimate_shift(f, g, 8, 16)


def test_shift_random_range_bit_exact(gpu, oracle):
    rng = Rng(77)
    for trial in range(12):
        f = textured_frame(128, 96, 8, 100 + trial)
        dx, dy = rng.next_below(21) - 10, rng.next_below(21) - 10
        g = cyclic_shift(f, dx, dy)
        s = gpu.estimate_shift(f, g, 16)
        assert (s.dx, s.dy) == (dx, dy)
        assert s == oracle.estimate_shift(f, g, 8, 16)  # confidence bit-identical


def test_shift_noise_blank_and_odd_sizes(gpu, oracle):
    a, b = random_frame(128, 128, 8, 11), random_frame(128, 128, 8, 12)
    s = gpu.estimate_shift(a, b, 16)
    assert s.confidence < 1.5
    assert s == oracle.estimate_shift(a, b, 8, 16)
    blank = np.full((64, 64), 50, np.uint16)
    s = gpu.estimate_shift(blank, blank, 8)
    assert (s.dx, s.dy) == (0, 0)
    assert s == oracle.estimate_shift(blank, blank, 8, 8)
    # non-power-of-two frames are edge-replicated into the FFT grid
    f = textured_frame(100, 72, 8, 3)
    g = cyclic_shift(f, -4, 2)
    assert gpu.estimate_shift(f, g, 12) == oracle.estimate_shift(f, g, 8, 12)


def test_shift_validation(gpu):
    from paper_2511_14419_b200.params import DataError, UsageError
    a = np.zeros((64, 64), np.uint16)
    with pytest.raises(DataError):
        gpu.estimate_shift(a, np.zeros((32, 32), np.uint16), 8)
    with pytest.raises(UsageError):
        gpu.estimate_shift(a, a, 16)


# ---------------------------------------------------------------- flow (flow.hpp)
def _flow_err(gu, gv, ou, ov):
    du, dv = gu.astype(np.float64) - ou, gv.astype(np.float64) - ov
    return max(np.abs(du).max(), np.abs(dv).max()), float(np.hypot(du, dv).mean())


@pytest.mark.parametrize("w,h,dx,dy,seed", [(96, 80, 2, 1, 21), (160, 160, 4, -3, 50),
                                             (128, 128, 0, 0, 7), (77, 65, -1, 2, 3)])
def test_flow_tolerance(gpu, oracle, w, h, dx, dy, seed):
    f = textured_frame(w, h, 8, seed)
    g = cyclic_shift(f, dx, dy) if (dx or dy) else textured_frame(w, h, 8, seed + 1)
    gu, gv = gpu.compute_flow(f, g)
    ou, ov = oracle.compute_flow(f, g, 8)
    mx, mean = _flow_err(gu, gv, ou, ov)
    assert mx <= FLOW_MAX_ABS and mean <= FLOW_MEAN_EPE, (mx, mean)


def test_flow_upsample_kernels_agree(tmp_path):
    """Exact 2:1 levels take k_upsample2 (nine loads per four outputs, 16-byte stores); the
    generic k_upsample (FROI_UPSAMPLE2=0) must give the same flow bit for bit -- both evaluate the
    same explicitly rounded expression.  256^2 (every level 2:1) and 200x152 (2:1 with a border)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "from paper_2511_14419_b200 import flowroi as F\n"
        "from fixtures import textured_frame, cyclic_shift\n"
        "out = []\n"
        "for w, h in ((256, 256), (200, 152)):\n"
        "    f = textured_frame(w, h, 8, 5); g = cyclic_shift(f, 3, -2)\n"
        "    u, v = F.compute_flow(f, g); out += [u.ravel(), v.ravel()]\n"
        "np.save(sys.argv[1], np.concatenate(out))\n"
    ) % (root, os.path.join(root, "tests"))
    outs = []
    for sel in ("1", "0"):
        p = str(tmp_path / f"u{sel}.npy")
        env = dict(os.environ, FROI_UPSAMPLE2=sel)
        subprocess.run([sys.executable, "-c", code, p], check=True, env=env, timeout=300)
        outs.append(np.load(p))
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))


def test_flow_identical_frames_exactly_zero(gpu):
    f = textured_frame(96, 80, 8, 21)
    u, v = gpu.compute_flow(f, f)
    assert not np.any(u) and not np.any(v)
    blank = np.full((64, 64), 100, np.uint16)
    u, v = gpu.compute_flow(blank, blank)
    assert not np.any(u) and not np.any(v)


def test_flow_pyramid_translation(gpu):
    f = textured_frame(160, 160, 8, 50)
    g = cyclic_shift(f, 4, -3)
    u, v = gpu.compute_flow(f, g)
    err = np.hypot(u[16:144, 16:144] - 4.0, v[16:144, 16:144] + 3.0).mean()
    assert err < 0.5


def test_flow_levels_and_16bit(gpu, oracle):
    from paper_2511_14419_b200.params import FlowParams
    f = (textured_frame(128, 96, 16, 4) >> 4).astype(np.uint16)
    g = cyclic_shift(f, 3, 1)
    for levels in (1, 2, 4):
        p = FlowParams(pyramid_levels=levels)
        from paper_2511_14419_b200.params import ExtractParams
        ep = ExtractParams(flow=p)
        gu, gv = gpu.compute_flow(f, g, p, depth=16)
        ou, ov = oracle.compute_flow(f, g, 16, ep)
        mx, mean = _flow_err(gu, gv, ou, ov)
        assert mx <= FLOW_MAX_ABS and mean <= FLOW_MEAN_EPE, (levels, mx, mean)


@pytest.mark.parametrize("scale,levels", [(0.6, 3), (0.75, 4), (0.5, 3)])
def test_flow_pyramid_scale(gpu, oracle, scale, levels):
    """Pyramids that are not 2:1 (resize_bilinear at a general factor, flow.hpp:277-298; the
    coarse-to-fine prior rescaled per axis, flow.hpp:318-337): the fp32 flow within the stated
    tolerance and the bit-exact mode identical to the reference, on an odd-sized frame pair."""
    from paper_2511_14419_b200.params import ExtractParams, FlowParams
    f = textured_frame(150, 118, 8, 17)
    g = cyclic_shift(f, 2, -3)
    p = FlowParams(pyramid_levels=levels, pyramid_scale=scale)
    ou, ov = oracle.compute_flow(f, g, 8, ExtractParams(flow=p))
    gu, gv = gpu.compute_flow(f, g, p)
    mx, mean = _flow_err(gu, gv, ou, ov)
    assert mx <= FLOW_MAX_ABS and mean <= FLOW_MEAN_EPE, (scale, mx, mean)
    xu, xv = gpu.compute_flow(f, g, p, exact=True)
    assert np.array_equal(xu, ou) and np.array_equal(xv, ov)


@pytest.mark.parametrize("levels,poly_n,poly_sigma,window,iters",
                         [(1, 5, 1.1, 15, 3), (2, 7, 1.5, 9, 2), (4, 5, 1.1, 5, 1), (3, 3, 0.8, 3, 4),
                          (3, 5, 1.1, 11, 3), (3, 7, 1.5, 13, 2)])
def test_flow_params_fp32(gpu, oracle, levels, poly_n, poly_sigma, window, iters):
    """The fp32 flow off the defaults: every box-window template (window 3..15 -> R 1..7), the
    runtime-radius polynomial expansion (poly_n 3 / 7), 1..4 levels and 1..4 iterations, on u8 and
    12-bit data -- within the stated tolerance of the fp64 reference."""
    from paper_2511_14419_b200.params import ExtractParams, FlowParams
    p = FlowParams(pyramid_levels=levels, poly_n=poly_n, poly_sigma=poly_sigma, window_size=window,
                   iterations=iters)
    ep = ExtractParams()
    ep.flow = p
    for depth in (8, 16):
        f = textured_frame(120, 104, depth, 9)
        if depth == 16:
            f = (f >> 4).astype(np.uint16)
        g = cyclic_shift(f, 2, -1)
        gu, gv = gpu.compute_flow(f, g, p, depth=depth)
        ou, ov = oracle.compute_flow(f, g, depth, ep)
        mx, mean = _flow_err(gu, gv, ou, ov)
        assert mx <= FLOW_MAX_ABS and mean <= FLOW_MEAN_EPE, (depth, levels, poly_n, window, iters, mx, mean)


def test_polynomial_expansion_kats(gpu, oracle):
    # constant -> A = b = 0, c = const (test_flow.cpp:66-79; fp32 tolerance)
    e = gpu.polynomial_expansion(np.full((32, 32), 0.42, np.float32))
    assert np.allclose(e[0, 4:28, 4:28], 0.42, rtol=1e-6)
    assert np.abs(e[1:, 4:28, 4:28]).max() < 1e-6
    # ramp -> bx = alpha (test_flow.cpp:81-93)
    x = np.arange(40, dtype=np.float64)[None, :].repeat(30, 0)
    e = gpu.polynomial_expansion((0.0125 * x).astype(np.float32))
    assert np.allclose(e[1, 3:27, 3:37], 0.0125, rtol=1e-5)
    # x^2 -> a11 = 1 (test_flow.cpp:114-124)
    e = gpu.polynomial_expansion((np.arange(32.0)[None, :] ** 2).repeat(32, 0).astype(np.float32))
    assert np.allclose(e[3, 4:28, 4:28], 1.0, rtol=1e-3)
    # against the fp64 reference on random data
    img = np.random.default_rng(31).random((48, 48))
    got = gpu.polynomial_expansion(img.astype(np.float32))
    want = oracle.polynomial_expansion(img)
    assert np.abs(got - want).max() < 2e-5


# ---------------------------------------------------------------- mask stage (roi.hpp)
def _oracle_flow_pair(oracle, w=96, h=80, seed=21, dx=2, dy=1):
    f = textured_frame(w, h, 8, seed)
    g = cyclic_shift(f, dx, dy)
    u, v = oracle.compute_flow(f, g, 8)
    return f, g, u, v


@pytest.mark.parametrize("source", [0, 1])
def test_saliency_bit_exact(gpu, oracle, source):
    f, g, u, v = _oracle_flow_pair(oracle)
    got = gpu.saliency(u, v, g, 0.7, source)
    want = oracle.saliency(u, v, g, 8, 0.7, source)
    assert np.array_equal(got, want)
    zero = np.zeros_like(u)
    assert np.array_equal(gpu.saliency(zero, zero, g), oracle.saliency(zero, zero, g, 8))
    const = np.full((32, 32), 100, np.uint16)
    z = np.zeros((32, 32), np.float32)
    assert not np.any(gpu.saliency(z, z, const))


def test_saliency_gradient_table_full_range(gpu, oracle):
    """8-bit frames take |grad I| from the context's table (every central-difference magnitude x
    every other, evaluated once with the restated glibc hypot): uniform-noise frames hit tens of
    thousands of distinct (|gx|, |gy|) entries, all below the 99th percentile compared exactly."""
    rng = np.random.default_rng(5)
    for shape, seed in (((256, 256), 1), ((200, 312), 2)):
        h, w = shape
        frame = rng.integers(0, 256, size=(h, w)).astype(np.uint8)
        u = rng.normal(0, 2, size=(h, w)).astype(np.float32)
        v = rng.normal(0, 2, size=(h, w)).astype(np.float32)
        for fw in (0.0, 0.7):
            got = gpu.saliency(u, v, frame, fw, 0, depth=8)
            want = oracle.saliency(u, v, frame, 8, fw, 0)
            assert np.array_equal(got, want)


def test_threshold_bit_exact(gpu, oracle):
    rng = Rng(23)
    perm = list(range(100))
    for i in range(99, 0, -1):
        j = rng.next_below(i + 1)
        perm[i], perm[j] = perm[j], perm[i]
    m = ((np.array(perm) + 1) / 101.0).reshape(10, 10)
    got = gpu.threshold_mask(m, 0.2)
    assert got.sum() == 20 and np.array_equal(got, oracle.threshold_mask(m, 0.2))
    two = (np.arange(100) % 2).astype(np.float64).reshape(10, 10)
    assert np.array_equal(gpu.threshold_mask(two, 0.5), oracle.threshold_mask(two, 0.5))
    assert gpu.threshold_mask(np.zeros((32, 32)), 0.2).sum() == 0
    gen = np.random.default_rng(3)
    for t in (0.05, 0.2, 0.5, 0.95):
        r = gen.random((100, 120))
        assert np.array_equal(gpu.threshold_mask(r, t), oracle.threshold_mask(r, t))
        # heavy ties: quantised values, admitted in row-major order
        q = np.floor(r * 7) / 7
        assert np.array_equal(gpu.threshold_mask(q, t), oracle.threshold_mask(q, t))
        # fewer positive values than the target: keep the positive ones
        sparse = np.where(r > 0.9, r, 0.0)
        assert np.array_equal(gpu.threshold_mask(sparse, 0.5), oracle.threshold_mask(sparse, 0.5))
    # widths that are whole 32-bit words take the fused path (threshold words written by the
    # collect pass, boundary-bin candidates settled afterwards): plain, heavy ties, sparse
    for shape in ((96, 128), (256, 256)):
        r = gen.random(shape)
        for t in (0.05, 0.2, 0.5):
            for m in (r, np.floor(r * 7) / 7, np.floor(r * 300) / 300, np.where(r > 0.9, r, 0.0)):
                assert np.array_equal(gpu.threshold_mask(m, t), oracle.threshold_mask(m, t)), (shape, t)


@pytest.mark.parametrize("ro,rc,min_area", [(1, 1, 20), (0, 0, 20), (1, 2, 12), (2, 3, 0), (1, 1, 1)])
def test_morph_cleanup_bit_exact(gpu, oracle, ro, rc, min_area):
    for trial in range(4):
        m = random_mask(70, 45, 0.35 + 0.1 * trial, 600 + trial)
        got = gpu.morph_cleanup(m, ro, rc, min_area)
        assert np.array_equal(got, oracle.morph_cleanup(m, ro, rc, min_area)), trial


def test_morph_kats(gpu):
    m = np.zeros((16, 16), np.uint8)
    m[8, 8] = 1
    assert gpu.morph_open(m, 1).sum() == 0
    sq = np.zeros((20, 20), np.uint8)
    sq[5:15, 5:15] = 1
    sq[9, 9] = 0
    c = gpu.morph_close(sq, 1)
    assert c[9, 9] == 1 and c.sum() == 100


def test_component_areas(gpu, oracle):
    for trial in range(6):
        m = random_mask(48 + 17 * trial, 48 + 9 * trial, 0.4, 700 + trial)
        assert np.array_equal(gpu.component_areas(m), oracle.component_areas(m))
    m = np.zeros((32, 32), np.uint8)
    m[2:5, 2:7] = 1
    m[20:25, 20:26] = 1
    out = gpu.morph_cleanup(m, 0, 0, 20)
    assert list(gpu.component_areas(out)) == [30]


@pytest.mark.parametrize("dx,dy", [(0, 0), (2, -1), (-3, 4)])
def test_mask_from_flow_bit_exact(gpu, oracle, dx, dy):
    f, g, u, v = _oracle_flow_pair(oracle, 128, 96, 5, 3, 2)
    got, st = gpu.mask_from_flow(u, v, g, dx, dy)
    want, dbg = oracle.mask_from_flow(u, v, g, 8, dx, dy)
    assert np.array_equal(got, want)
    assert st["mask_count"] == int(want.sum())


def test_temporal_ensemble(gpu):
    ms = np.zeros((3, 16, 16), np.uint8)
    ms[0, 2, 2] = ms[1, 8, 8] = ms[2, 14, 14] = 1
    u = gpu.temporal_ensemble(ms, 1, 1)
    assert u.sum() == 3 and u[2, 2] and u[8, 8] and u[14, 14]
    assert np.array_equal(gpu.temporal_ensemble(ms, 1, 0), ms[1])
