"""Throughput on the other BASELINE configurations (SURVEY.md §8d asks for C2 and C4 beside C3).

  python profiles/tools/config_tput.py [C2 C3 C4 ...]      (on the GPU box)

Per config, one JSON line: frames/s device-resident (froi_extract_wells_device, CUDA events on
the context stream, two lanes), end to end through froi_extract_wells (pinned frames in, pinned
PBM masks out), and the reference compiled in place (oracle/_ref extract_roi, every host thread)
on a bounded sample of the same well.  Synthetic frames (gen/synth.c), the config's own params.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2511_14419_b200 import flowroi, synth  # noqa: E402
from paper_2511_14419_b200.params import CFrameStats  # noqa: E402


def run(name: str, steps: int = 5, warmup: int = 3, ref_frames: int = 0) -> dict:
    cfg = synth.config(name)
    F, W, H = cfg.n_frames, cfg.width, cfg.height
    dt = np.uint8 if cfg.sample_bytes == 1 else np.uint16
    host = torch.empty((F, H, W), dtype=torch.uint8 if dt == np.uint8 else torch.int16, pin_memory=True)
    hv = host.numpy().view(dt)
    synth.well_frames(cfg, 0, F, out=hv)
    dev = host.cuda()
    SB = (W + 7) // 8
    dmask = torch.empty((F, H, SB), dtype=torch.uint8, device="cuda")
    hmask = torch.empty((F, H, SB), dtype=torch.uint8, pin_memory=True)
    ctx = flowroi.Context(W, H, cfg.depth, cfg.params)
    s = torch.cuda.ExternalStream(ctx.stream())
    for _ in range(warmup):
        ctx.extract_wells_device(dev.data_ptr(), 1, F, dmask.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        ctx.extract_wells_device(dev.data_ptr(), 1, F, dmask.data_ptr())
    e1.record(s)
    torch.cuda.synchronize()
    dev_fps = steps * F / (e0.elapsed_time(e1) / 1e3)
    stats = (CFrameStats * F)()
    for _ in range(2):
        ctx.extract_wells_into(hv[None], hmask.numpy(), stats)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(steps):
        ctx.extract_wells_into(hv[None], hmask.numpy(), stats)
        _ = hmask[0, 0, 0].item()
    e1.record(s)
    torch.cuda.synchronize()
    e2e_fps = steps * F / (e0.elapsed_time(e1) / 1e3)
    same = bool(torch.equal(dmask.cpu(), hmask))
    ctx.close()
    out = {"config": name, "frames": F, "shape": [H, W], "depth": cfg.depth,
           "pyramid_levels": cfg.params.flow.pyramid_levels, "device_frames_per_s": round(dev_fps, 1),
           "e2e_frames_per_s": round(e2e_fps, 1), "device_equals_e2e_masks": same}
    if ref_frames:
        from oracle.oracle_py import Oracle, reference_available
        if reference_available():
            cores = os.cpu_count() or 1
            fr = hv[:ref_frames].copy()
            t0 = time.perf_counter()
            Oracle("reference").extract_roi(fr, cfg.depth, cfg.params, workers=cores)
            t = time.perf_counter() - t0
            out["reference_frames_per_s"] = round(ref_frames / t, 3)
            out["reference_sample"] = f"{ref_frames} frames of well 0, workers={cores}, {t:.1f} s"
            out["e2e_speedup"] = round(e2e_fps / (ref_frames / t), 1)
    return out


if __name__ == "__main__":
    names = sys.argv[1:] or ["C2", "C3", "C4"]
    cores = os.cpu_count() or 1
    ref = {"C2": min(64, 8 * cores + 1), "C3": min(450, 8 * cores + 1), "C4": min(128, 2 * cores + 1)}
    for n in names:
        print(json.dumps(run(n, ref_frames=ref.get(n, 0))), flush=True)
