"""Runs a fixed set of GPU cases and saves their masks (helper of test_gpu_checked.py).

    FROI_LIB=<lib> python tests/_checked_runner.py OUT.npz

Cases: C1 (512^2, one pair); a two-well 256^2 sequence of 13 frames on two lanes with 4-pair
batches (multi-batch, lane alternation, egress ring); the same through the host entry with pinned
PBM output; a 12-bit 256^2 sequence; and a low-threshold case that exercises partial tie
admission and the CCL area filter; C1 and the two wells through the bit-exact flow mode.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2511_14419_b200 import flowroi as F, synth  # noqa: E402


def main(out):
    res = {}
    cfg = synth.config("C1")
    res["c1"] = F.extract_roi(synth.well_frames(cfg, 0, 2), cfg.params)
    c2 = synth.scaled(synth.config("C2"), width=256, height=256, n_cells=20)
    frames = np.stack([synth.well_frames(synth.scaled(c2, seed=40 + w), 0, 13) for w in range(2)])
    for mp in (2, 3, 4, 32):
        for lanes in (1, 2):
            ctx = F.Context(256, 256, 8, c2.params, device=0, max_pairs=mp)
            ctx.set_lanes(lanes)
            m, _ = ctx.extract_wells(frames, layout="pbm")
            res[f"wells_mp{mp}_l{lanes}"] = m
            if mp == 4:  # the intra-batch fork off: same bytes
                ctx.set_fork(False)
                m, _ = ctx.extract_wells(frames, layout="pbm")
                res[f"wells_mp{mp}_l{lanes}_nofork"] = m
            ctx.close()
    c4 = synth.scaled(synth.config("C4"), width=256, height=256, n_cells=30)
    res["u16"] = F.extract_roi(synth.well_frames(c4, 0, 3), c4.params, depth=16)
    p = c2.params.copy()
    p.roi.roi_threshold = 0.05
    p.roi.min_area = 40
    res["lowthr"] = F.extract_roi(frames[0, :4], p)
    # the bit-exact flow mode: C1, and the two wells multi-batch on two lanes
    res["c1_exact"] = F.extract_roi(synth.well_frames(cfg, 0, 2), cfg.params, exact_flow=True)
    ctx = F.Context(256, 256, 8, c2.params, device=0, max_pairs=3)
    ctx.set_flow_exact(True)
    m, _ = ctx.extract_wells(frames, layout="pbm")
    res["exact_wells_mp3"] = m
    ctx.close()
    np.savez_compressed(out, **res)


if __name__ == "__main__":
    main(sys.argv[1])
