"""Generates tests/golden/golden_small.npz from the REFERENCE compiled in place
(oracle/_ref/libfroi_ref.so built from /root/reference by oracle/Makefile).

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
The fixtures pin the C restatement (oracle/froi_oracle.c) and the Python fixture restatement
(tests/fixtures.py) on machines without the reference tree.
"""
import ctypes
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

from fixtures import cyclic_shift, textured_frame  # noqa: E402
from oracle.oracle_py import Oracle, ensure_built  # noqa: E402
from paper_2511_14419_b200.params import ExtractParams  # noqa: E402


def main():
    ensure_built(reference=True)
    ref = Oracle("reference")
    out = {}
    # Rng streams (rng.hpp)
    n = 64
    u64 = np.zeros(n, np.uint64)
    nrm = np.zeros(n, np.float64)
    ref.lib.ref_rng_stream.restype = None
    ref.lib.ref_rng_stream(ctypes.c_uint64(909), n, ctypes.c_void_p(u64.ctypes.data),
                           ctypes.c_void_p(nrm.ctypes.data))
    out["rng_seed"] = np.array(909)
    out["rng_u64"] = u64
    out["rng_normal"] = nrm
    # denoise, u8 and 12-bit-in-16
    f8 = textured_frame(48, 40, 8, 909)
    f16 = (textured_frame(33, 21, 16, 8) >> 4).astype(np.uint16)
    out["den_in8"], out["den_out8"] = f8, ref.denoise(f8, 8)
    out["den_in16"], out["den_out16"] = f16, ref.denoise(f16, 16)
    # registration
    a = textured_frame(128, 96, 8, 100)
    b = cyclic_shift(a, 3, -2)
    s = ref.estimate_shift(a, b, 8, 16)
    out["reg_a"], out["reg_b"] = a, b
    out["reg_shift"] = np.array([s.dx, s.dy, s.confidence])
    # flow
    f = textured_frame(96, 80, 8, 21)
    g = cyclic_shift(f, 2, 1)
    u, v = ref.compute_flow(f, g, 8)
    out["flow_a"], out["flow_b"], out["flow_u"], out["flow_v"] = f, g, u, v
    # saliency / threshold / cleanup on that flow
    sal = ref.saliency(u, v, g, 8)
    out["sal"] = sal
    thr = ref.threshold_mask(sal, 0.2)
    out["thr"] = thr
    out["clean"] = ref.morph_cleanup(thr, 1, 1, 20)
    # a whole small sequence from the reference generator (synthetic.hpp)
    frames, truth, xy, radii = ref.generate_synthetic(n_cells=3, n_frames=4, width=96, height=96,
                                                      seed=55)
    masks, shifts, fracs = ref.extract_roi(frames, 8, ExtractParams())
    out["seq_frames"], out["seq_masks"] = frames, masks
    out["seq_shifts"] = np.array([[s.dx, s.dy, s.confidence] for s in shifts])
    out["seq_fracs"] = fracs
    np.savez_compressed(os.path.join(HERE, "golden_small.npz"), **out)
    print("wrote", os.path.join(HERE, "golden_small.npz"))


if __name__ == "__main__":
    main()
