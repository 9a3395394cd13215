"""Workloads for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

  python profiles/tools/sanitize_cases.py c1      C1: one 512^2 u8 pair, default parameters
  python profiles/tools/sanitize_cases.py lanes   two execution lanes, several batches
                                                  (max_pairs 4, 13 frames of 256^2, two wells),
                                                  host entry with pinned PBM read-back, then the
                                                  device entry; both outputs must agree
  python profiles/tools/sanitize_cases.py u16     C4-style 12-bit frames (256^2, depth 16, L = 5
                                                  is capped by the 32 px rule), 3 frames

Each case exits non-zero if the GPU result differs between the entry points it runs; the
sanitizer's own report decides the race / memory verdict (profiles/r02_sanitizer.md).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2511_14419_b200 import flowroi as F, synth  # noqa: E402
from paper_2511_14419_b200.params import CFrameStats  # noqa: E402


def case_c1():
    cfg = synth.config("C1")
    frames = synth.well_frames(cfg, 0, 2)
    m = F.extract_roi(frames, cfg.params)
    print("c1 mask fraction", float(m.mean()))


def case_lanes():
    import ctypes
    cfg = synth.scaled(synth.config("C2"), width=256, height=256, n_cells=20)
    n, nw = 13, 2
    frames = np.stack([synth.well_frames(synth.scaled(cfg, seed=40 + w), 0, n) for w in range(nw)])
    ctx = F.Context(256, 256, 8, cfg.params, device=0, max_pairs=4)
    ctx.set_lanes(2)
    a, st = ctx.extract_wells(frames, layout="pbm")
    # host entry with pinned output (per-batch read-back on the D2H stream)
    import torch
    pin = torch.empty(a.shape, dtype=torch.uint8, pin_memory=True)
    hin = torch.empty(frames.shape, dtype=torch.uint8, pin_memory=True)
    hin.numpy()[:] = frames
    stats = (CFrameStats * (nw * n))()
    ctx.extract_wells_into(hin.numpy(), pin.numpy(), stats)
    # device entry
    dfr = torch.from_numpy(frames).cuda()
    dm = torch.empty(a.shape, dtype=torch.uint8, device="cuda")
    ctx.extract_wells_device(dfr.data_ptr(), nw, n, dm.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(a, pin.numpy()), "pinned host entry differs"
    assert np.array_equal(a, dm.cpu().numpy()), "device entry differs"
    ctx.set_lanes(1)
    b, _ = ctx.extract_wells(frames, layout="pbm")
    assert np.array_equal(a, b), "one lane differs from two lanes"
    ctx.close()
    print("lanes ok", a.shape)


def case_u16():
    cfg = synth.scaled(synth.config("C4"), width=256, height=256, n_cells=30)
    frames = synth.well_frames(cfg, 0, 3)
    m = F.extract_roi(frames, cfg.params, depth=16)
    print("u16 mask fraction", float(m.mean()))


if __name__ == "__main__":
    {"c1": case_c1, "lanes": case_lanes, "u16": case_u16}[sys.argv[1]]()
