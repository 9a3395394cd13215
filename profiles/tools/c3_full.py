"""The whole C3 configuration (64 wells x 450 frames, 28,800 masks, 30.2 GB of 1024^2 u8 frames)
through the public host API on one GPU (run on the GPU box):

  python profiles/tools/c3_full.py [wells] [config]      (config C3 by default; C4: 16 x 128 2048^2 u16)

Each well is rendered into pinned memory (gen/synth.c, the bench's generator) while the previous
well runs on the GPU; each call is froi_extract_wells (pinned frames in, PBM masks out, H2D and D2H
inside the call).  Prints one JSON line: total GPU-call time, masks/s, and per-well mask-fraction
and shift statistics (a sanity summary of all 28,800 masks).
"""
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2511_14419_b200 import flowroi, synth  # noqa: E402
from paper_2511_14419_b200.params import CFrameStats  # noqa: E402

cfg = synth.config(sys.argv[2] if len(sys.argv) > 2 else "C3")
nw = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.n_wells
F, W, H = cfg.n_frames, cfg.width, cfg.height
u16 = cfg.sample_bytes == 2
bufs = [torch.empty((F, H, W), dtype=torch.int16 if u16 else torch.uint8, pin_memory=True) for _ in range(2)]
masks = torch.empty((F, H, (W + 7) // 8), dtype=torch.uint8, pin_memory=True)
ctx = flowroi.Context(W, H, cfg.depth, cfg.params)
view = (lambda t: t.numpy().view(np.uint16)) if u16 else (lambda t: t.numpy())
stats = (CFrameStats * F)()
synth.well_frames(cfg, 0, F, out=view(bufs[0]))
call_s, fracs, shifted, set_px = 0.0, [], 0, 0
for w in range(nw):
    cur = view(bufs[w % 2])
    th = None
    if w + 1 < nw:  # render the next well while this one runs
        th = threading.Thread(target=synth.well_frames, args=(cfg, w + 1, F),
                              kwargs={"out": view(bufs[(w + 1) % 2])})
        th.start()
    t0 = time.perf_counter()
    ctx.extract_wells_into(cur[None], masks.numpy(), stats)
    call_s += time.perf_counter() - t0
    fr = np.array([stats[t].raw_fraction for t in range(F)])
    fracs.append((float(fr.mean()), float(fr.min()), float(fr.max())))
    shifted += sum(1 for t in range(1, F) if stats[t].dx or stats[t].dy)
    set_px += sum(int(stats[t].mask_count) for t in range(F))
    if th:
        th.join()
ctx.close()
out = {"config": cfg.name, "wells": nw, "frames": nw * F, "masks": nw * F,
       "input_gb": nw * F * W * H * cfg.sample_bytes / 1e9,
       "gpu_call_s": round(call_s, 3), "masks_per_s": round(nw * F / call_s, 1),
       "raw_fraction_mean": round(float(np.mean([f[0] for f in fracs])), 5),
       "raw_fraction_min": round(float(min(f[1] for f in fracs)), 5),
       "raw_fraction_max": round(float(max(f[2] for f in fracs)), 5),
       "pairs_with_nonzero_shift": shifted, "mask_pixels_set": set_px,
       "note": "host-clock time of the extract_wells calls only (well rendering overlapped, not counted)"}
print(json.dumps(out), flush=True)
