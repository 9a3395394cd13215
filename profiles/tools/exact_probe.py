"""One 65-frame C3 batch through the bit-exact flow mode (for ncu launch lists of k64_*).
  ncu --metrics gpu__time_duration.sum -k regex:k64 python profiles/tools/exact_probe.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2511_14419_b200 import flowroi, synth  # noqa: E402

cfg = synth.config("C3")
F = int(sys.argv[1]) if len(sys.argv) > 1 else 65
frames = synth.well_frames(cfg, 0, F)
ctx = flowroi.Context(1024, 1024, 8, cfg.params)
ctx.set_lanes(1)
ctx.set_flow_exact(True)
m, _ = ctx.extract_wells(frames[None])
print("mask pixels", int(m.sum()))
ctx.close()
