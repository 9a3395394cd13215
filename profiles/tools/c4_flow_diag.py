"""Where the C4 flow differs most from the fp64 oracle (run on the GPU box).
Prints, per pair of two C4 wells x 8 frames, max |d|, the number of pixels above 1e-2 / 5e-3, and
for the worst pixel the GPU / oracle (u, v) there and the oracle's local spread."""
import multiprocessing
import os
import sys
from concurrent.futures import ProcessPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2511_14419_b200 import flowroi as F, synth  # noqa: E402


def oracle_flow(args):
    from oracle.oracle_py import Oracle
    a, b, depth, params = args
    return Oracle("port").compute_flow(a, b, depth, params)


def shifted(f, dx, dy):
    h, w = f.shape
    return f[np.clip(np.arange(h) + dy, 0, h - 1)][:, np.clip(np.arange(w) + dx, 0, w - 1)]


def main():
    cfg = synth.config("C4")
    jobs, gfl, tags = [], [], []
    for well in (0, 5):
        fr = synth.well_frames(cfg, well, 8)
        den = [F.denoise(fr[t], cfg.params, depth=16) for t in range(8)]
        for t in range(1, 8):
            s = F.estimate_shift(den[t - 1], den[t], cfg.params.max_shift, depth=16)
            dx, dy = (s.dx, s.dy) if s.confidence >= 1.5 else (0, 0)
            nxt = shifted(den[t], dx, dy)
            gfl.append(F.compute_flow(den[t - 1], nxt, cfg.params, depth=16))
            jobs.append((den[t - 1], nxt, 16, cfg.params))
            tags.append((well, t, dx, dy))
    with ProcessPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 1),
                             mp_context=multiprocessing.get_context("spawn")) as ex:
        ofl = list(ex.map(oracle_flow, jobs))
    for tag, (gu, gv), (ou, ov) in zip(tags, gfl, ofl):
        d = np.maximum(np.abs(gu - ou), np.abs(gv - ov))
        y, x = np.unravel_index(np.argmax(d), d.shape)
        win = (slice(max(0, y - 2), y + 3), slice(max(0, x - 2), x + 3))
        print(tag, f"max {d.max():.4f} at ({x},{y}); >1e-2: {int((d > 1e-2).sum())}, >5e-3: {int((d > 5e-3).sum())}, "
              f"mean EPE {np.hypot(gu - ou, gv - ov).mean():.2e}; gpu ({gu[y, x]:.4f},{gv[y, x]:.4f}) "
              f"oracle ({ou[y, x]:.4f},{ov[y, x]:.4f}); oracle local u range {np.ptp(ou[win]):.4f} v range {np.ptp(ov[win]):.4f}; "
              f"|flow| {np.hypot(ou[y, x], ov[y, x]):.2f}", flush=True)


if __name__ == "__main__":
    main()
