"""Flow precision of several library builds on every pair of one well vs the fp64 oracle.

  python profiles/tools/flow_precision_sweep.py CONFIG WELL NFRAMES lib1.so [lib2.so ...]

Denoise / registration come from the first library (bit-exact in every build); each library's
froi_compute_flow then runs on the same registered pairs (loaded side by side with ctypes), and
the oracle flow of each pair is computed once on all host cores.  Prints per library: max |d|
over the well, p99 over pairs, mean EPE max, pixels above 1e-2.
"""
import ctypes
import multiprocessing
import os
import sys
from concurrent.futures import ProcessPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402


def oracle_flow(args):
    from oracle.oracle_py import Oracle
    a, b, depth, params = args
    u, v = Oracle("port").compute_flow(a, b, depth, params)
    return u.astype(np.float64), v.astype(np.float64)


def shifted(f, dx, dy):
    h, w = f.shape
    return f[np.clip(np.arange(h) + dy, 0, h - 1)][:, np.clip(np.arange(w) + dx, 0, w - 1)]


def main():
    from paper_2511_14419_b200 import flowroi as F, synth
    from paper_2511_14419_b200.params import ExtractParams
    cname, well, nfr = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    libs = sys.argv[4:]
    cfg = synth.config(cname)
    depth = cfg.depth
    fr = synth.well_frames(cfg, well, nfr)
    den = [F.denoise(fr[t], cfg.params, depth=depth) for t in range(nfr)]
    pairs = []
    for t in range(1, nfr):
        s = F.estimate_shift(den[t - 1], den[t], cfg.params.max_shift, depth=depth)
        dx, dy = (s.dx, s.dy) if s.confidence >= 1.5 else (0, 0)
        pairs.append((np.ascontiguousarray(den[t - 1], dtype=np.uint16),
                      np.ascontiguousarray(shifted(den[t], dx, dy), dtype=np.uint16)))
    h, w = pairs[0][0].shape
    ep = ExtractParams() if cfg.params is None else cfg.params.copy()
    ep.max_shift = max(1, min(ep.max_shift, min(w, h) // 4 - 1))
    cp = ep.to_c()
    ctxs = []
    for lib in libs:
        L = ctypes.CDLL(os.path.abspath(lib))
        L.froi_ctx_create.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
        L.froi_compute_flow.argtypes = [ctypes.c_void_p] * 5
        c = ctypes.c_void_p()
        assert L.froi_ctx_create(0, ctypes.byref(cp), w, h, depth, 2, ctypes.byref(c)) == 0
        ctxs.append((lib, L, c))
    stats = {lib: [] for lib in libs}
    chunk = 32
    with ProcessPoolExecutor(max_workers=os.cpu_count() or 1,
                             mp_context=multiprocessing.get_context("spawn")) as ex:
        for k0 in range(0, len(pairs), chunk):
            sub = pairs[k0:k0 + chunk]
            ofl = list(ex.map(oracle_flow, [(a, b, depth, ep) for a, b in sub]))
            for (a, b), (ou, ov) in zip(sub, ofl):
                for lib, L, c in ctxs:
                    u = np.empty((h, w), np.float32)
                    v = np.empty((h, w), np.float32)
                    assert L.froi_compute_flow(c, a.ctypes.data, b.ctypes.data, u.ctypes.data, v.ctypes.data) == 0
                    d = np.maximum(np.abs(u - ou), np.abs(v - ov))
                    stats[lib].append((float(d.max()), float(np.hypot(u - ou, v - ov).mean()), int((d > 1e-2).sum())))
    for lib in libs:
        a = np.array(stats[lib])
        print(f"{os.path.basename(lib):22s} {cname} well {well} x {nfr}: max |d| {a[:, 0].max():.4f} "
              f"(pair {int(a[:, 0].argmax()) + 1}), p99 {np.percentile(a[:, 0], 99):.4f}, median {np.median(a[:, 0]):.4f}; "
              f"mean EPE max {a[:, 1].max():.2e}; pairs > 1e-2: {int((a[:, 0] > 1e-2).sum())}, "
              f"pixels > 1e-2: {int(a[:, 2].sum())}", flush=True)


if __name__ == "__main__":
    main()
