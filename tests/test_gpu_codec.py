"""Codec side on the GPU: reversible 5/3 DWT (dwt.hpp:113-171) and the RoI
coefficient masks (map_mask_to_subbands, codec.hpp:152-171), bit-exact against the oracle, whose
restatement is pinned to the reference in tests/test_oracle_pin.py."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("w,h,depth,levels", [(64, 64, 8, 5), (33, 17, 8, 3), (160, 96, 16, 4),
                                              (255, 129, 16, 5), (1024, 1024, 8, 5), (8, 8, 8, 3)])
def test_dwt_bit_exact(gpu, oracle, w, h, depth, levels):
    from paper_2511_14419_b200 import flowroi
    rng = np.random.default_rng(w + 3 * h + depth)
    frame = rng.integers(0, 1 << depth, (h, w), dtype=np.uint16)
    c = flowroi.dwt_forward(frame, levels, depth=depth)
    assert np.array_equal(c, oracle.dwt_forward(frame, depth, levels))
    assert np.array_equal(flowroi.dwt_inverse(c, levels, depth=depth), frame)
    # out-of-range coefficients clamp like clamp_to_depth
    c2 = c.copy()
    c2[0, 0] += 1 << 20
    assert np.array_equal(flowroi.dwt_inverse(c2, levels, depth=depth), oracle.dwt_inverse(c2, depth, levels))


@pytest.mark.parametrize("w,h,levels", [(64, 64, 5), (33, 17, 3), (1024, 1024, 5), (161, 97, 4)])
def test_map_mask_to_subbands_bit_exact(gpu, oracle, w, h, levels):
    from paper_2511_14419_b200 import flowroi
    rng = np.random.default_rng(w * h)
    for density in (0.0, 0.002, 0.05, 0.5):
        mask = (rng.random((h, w)) < density).astype(np.uint8)
        got = flowroi.map_mask_to_subbands(mask, levels)
        want = oracle.map_mask_to_subbands(mask, levels)
        assert all(np.array_equal(a, b) for a, b in zip(got, want))


def test_dwt_device_batch_and_validation(gpu, oracle):
    import torch
    from paper_2511_14419_b200 import _native, flowroi
    from paper_2511_14419_b200.params import DataError, ExtractParams, UsageError
    n, w, h, levels = 5, 96, 64, 4
    frames = np.stack([np.random.default_rng(k).integers(0, 256, (h, w), dtype=np.uint8) for k in range(n)])
    ep = ExtractParams()
    ep.max_shift = 8
    ctx = flowroi.Context(w, h, 8, ep)
    d_f = torch.from_numpy(frames).cuda()
    d_c = torch.empty((n, h, w), dtype=torch.int32, device="cuda")
    _native.check(_native.lib.froi_dwt_forward_device(ctx.handle, d_f.data_ptr(), n, levels, d_c.data_ptr()))
    got = d_c.cpu().numpy()
    for k in range(n):
        assert np.array_equal(got[k], oracle.dwt_forward(frames[k].astype(np.uint16), 8, levels))
    with pytest.raises(UsageError):
        flowroi.dwt_forward(frames[0], 0)
    with pytest.raises(DataError):
        flowroi.dwt_forward(frames[0], 7)  # 64 < 2^7
