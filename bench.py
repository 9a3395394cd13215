#!/usr/bin/env python
"""bench.py — RoI-mask frames/s of the B200 extract_roi stage on BASELINE config 3.

Workload (BASELINE.json configs[2], "C3"): wells of 450 frames, 1024x1024 uint8, each well
independently seeded with U{50..400} cells, wells sharded w -> rank (w mod N).  One *step* is one
complete well per rank (450 frames -> 449 adjacent pairs -> 450 masks) run through the stage
entry; step i of rank r processes C3 well (i*N + r) mod 64, so per-GPU work per step is fixed
("weak" scaling, no collective on the data path).  Frames are synthetic (gen/synth.c, seeded per
well); one well is 472 MB, far above the 126 MB L2, so no flush is needed between steps.

Legs of one run (rank 0 prints ONE JSON line):
  value      frames/s with the frames already resident in HBM (froi_extract_wells_device), timed
             with CUDA events on the context stream, max over ranks;
  e2e        the same metric through the public host API (froi_extract_wells: pinned host frames
             -> PBM masks in pinned host memory; H2D and D2H inside the timed region);
  roofline   the fused flow kernel (k_flow_iter): algorithmic bytes
             divided by its event-timed duration, against MEASURED_PEAKS.json hbm_gbs;
  cpu_baseline  the reference compiled in place (oracle/_ref, or the C restatement) on a bounded
             sample of the same wells with all host threads, rank 0 only.
`--impl reference` times only the reference CPU path (rank 0; other ranks exit 0).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RoI-mask frames/sec (1024² frame pairs) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "frames/s"
C3_WELLS = 64
W = H = 1024


def peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "source": "fallback"}


def levels_geometry(w: int, h: int, levels: int = 3) -> list:
    out = [(w, h)]
    while len(out) < levels:
        tw, th = int(out[-1][0] * 0.5), int(out[-1][1] * 0.5)
        if tw < 32 or th < 32:
            break
        out.append((tw, th))
    return out


def model_bytes_per_pair(w: int, h: int, b: int = 1, levels: int = 3) -> dict:
    """SURVEY.md App. C canonical algorithmic bytes per adjacent pair, per stage."""
    geo = levels_geometry(w, h, levels)
    n = [x * y for x, y in geo]
    N = n[0]
    S = sum(n) / N
    P = 1 << (max(w, h) - 1).bit_length()
    P = P * P
    pyr = b * N + (4 * n[1] if len(n) > 1 else 0) + sum(4 * n[l - 1] + 4 * n[l] for l in range(2, len(n)))
    st = {
        "denoise": 2 * b * N,
        "registration": b * N + 32 * P,
        "pyramid": 2 * pyr,
        "expansion": 2 * (b * N + 20 * N + 24 * (S - 1) * N),
        "flow": 160 * S * N + 8 * (S - 1) * N,
        "mask": 3 * (8 + b) * N + 8.25 * N,
    }
    st["total"] = sum(st.values())
    return st


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def init_dist(world: int, backend: str):
    if world <= 1:
        return None
    import torch.distributed as dist
    if not dist.is_initialized():
        dist.init_process_group(backend)
    return dist


def reduce_max(dist, x: float, device) -> float:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(dist, x: float, device) -> float:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


def free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def launch_ranks(n: int, argv: list[str], need_gpus: bool = True) -> int:
    """`bench.py --gpus N` without an external launcher: one process per GPU (RANK / LOCAL_RANK /
    WORLD_SIZE / MASTER_* set as torchrun would, rendezvous on 127.0.0.1).  Refuses to run when
    fewer than N GPUs are visible instead of measuring fewer.  Returns the worst exit code."""
    if need_gpus:
        import torch
        vis = torch.cuda.device_count()
        if vis < n:
            print(f"bench.py: --gpus {n} but only {vis} CUDA device(s) are visible", file=sys.stderr)
            return 3
    port = free_port()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(n), LOCAL_RANK=str(r),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + argv, env=env))
    rcs = [p.wait() for p in procs]
    return max((abs(rc) for rc in rcs), default=0)


def bind_numa(local: int) -> str:
    """Pins this rank to the host cores of its GPU's NUMA node (before the pinned host buffers
    are first touched, so they land in local memory).  Best effort: returns what was done."""
    try:
        import pynvml
        pynvml.nvmlInit()
        bus = pynvml.nvmlDeviceGetPciInfo(pynvml.nvmlDeviceGetHandleByIndex(local)).busId
        bus = bus.decode() if isinstance(bus, bytes) else bus
        dev = bus.lower()[-12:]  # dddd:bb:dd.f
        with open(f"/sys/bus/pci/devices/{dev}/numa_node") as f:
            node = int(f.read().strip())
        if node < 0:
            return "no NUMA affinity reported"
        with open(f"/sys/devices/system/node/node{node}/cpulist") as f:
            spec = f.read().strip()
        cpus = set()
        for part in spec.split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        os.sched_setaffinity(0, cpus)
        return f"node {node} ({len(cpus)} cores)"
    except Exception as e:  # pragma: no cover - depends on the host
        return f"not bound ({type(e).__name__})"


def wells_for(rank: int, world: int, steps: int) -> list[int]:
    """C3 well of each step of this rank: well (i*N + r) mod 64."""
    return [(i * world + rank) % C3_WELLS for i in range(steps)]


# ------------------------------------------------------------------ CPU reference leg
def sample_frames(cores: int) -> int:
    """Frames of a C3 well per CPU sample: 8 pairs per host thread (8c + 1), at most one well."""
    return max(3, min(8 * cores + 1, 450))


def cpu_reference(frames_per_sample: int, seconds_budget: float, steps: int, warmup: int,
                  threads: int | None = None) -> dict:
    """Times the reference CPU extract_roi (oracle/_ref when built, else the C restatement) on
    bounded samples of C3 wells with every host thread."""
    from oracle.oracle_py import Oracle, reference_available
    from paper_2511_14419_b200 import synth
    if not reference_available() and not os.environ.get("FROI_BENCH_ALLOW_PORT"):
        # the reference arm must time the reference itself (oracle/_ref, compiled in place from
        # /root/reference by oracle/Makefile); timing the restatement instead would void it
        raise SystemExit("bench.py: oracle/_ref/libfroi_ref.so is missing (build it here with "
                         "`make -C oracle ref`); refusing to time the C restatement as the reference")
    kind = "reference" if reference_available() else "port"
    # every host core: undo the rank's NUMA pinning (bind_numa) for the reference's own threads
    try:
        os.sched_setaffinity(0, range(os.cpu_count() or 1))
    except OSError:
        pass
    o = Oracle(kind)
    cfg = synth.config("C3")
    cores = threads or os.cpu_count() or 1
    times, masks = [], 0
    for i in range(warmup + steps):
        fr = synth.well_frames(cfg, well=i % C3_WELLS, n_frames=frames_per_sample)
        t0 = time.perf_counter()
        o.extract_roi(fr, 8, cfg.params, workers=cores)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
            masks += frames_per_sample
    total = sum(times)
    return {"value": masks / total, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{steps} C3 wells x {frames_per_sample} frames (1024^2 u8), extract_roi "
                      f"workers={cores}, {total:.1f} s", "seconds": total}


def run_reference(args) -> None:
    rank, world, local = dist_env()
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    # 8 pairs per host thread per step (~2.5 core-s per 1024^2 pair): with n = 8c + 1 frames the
    # reference's static partition (parallel.hpp:33-46) keeps every thread busy in the pair loop
    # and 15 of 16 in the denoise loop; a (c + 1)-frame sample left 7 of 16 idle in denoise
    frames = sample_frames(cores)
    r = cpu_reference(frames, 0, args.steps, args.warmup, cores)
    line = {
        "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * r["seconds"] / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C3: 64 wells x 450 frames, 1024x1024 u8 (one full well per "
                               "rank per step, well (i*N+r) mod 64)",
                   "sample": f"bounded CPU sample: {frames} frames of a C3 well per step",
                   "frames_per_step": frames, "parallelism": f"host threads={cores}",
                   "params": "ExtractParams{} defaults (pyramid 3, window 15, threshold 0.2)"},
        "impl": "reference",
        "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": cores, "kind": r["kind"],
                         "sample": r["sample"]},
        "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ launcher self-test (CPU)
def run_selftest(args) -> None:
    """The multi-rank plumbing of the GPU leg without a GPU (gloo): each rank takes its wells,
    reports a per-rank device time, and rank 0 prints the max-over-ranks time, the whole-job
    frame count and every rank's wells.  tests/test_multirank_cpu.py drives it through
    launch_ranks exactly as `bench.py --gpus N` does on a GPU box."""
    import torch
    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    dist = init_dist(world, "gloo")
    dev = torch.device("cpu")
    wells = wells_for(rank, world, args.warmup + args.steps)[args.warmup:]
    ms = reduce_max(dist, 100.0 + 10.0 * rank, dev)
    frames = reduce_sum(dist, float(len(wells) * args.frames), dev)
    allw = [None] * world if dist is not None else [wells]
    if dist is not None:
        dist.all_gather_object(allw, wells)
    if rank == 0:
        print(json.dumps({"selftest": True, "n_gpus": world, "ms_max": ms, "frames": frames,
                          "value": frames / (ms / 1000.0), "wells": allw}), flush=True)
    if dist is not None:
        dist.destroy_process_group()


# ------------------------------------------------------------------ drop-in leg
def run_dropin(frames: np.ndarray, steps: int, warmup: int, ref_pixels) -> dict | None:
    """Times oracle/_ref/dropin_bench: flowroi_gpu::extract_roi (include/froi/flowroi_gpu.hpp)
    over the reference's own types — a Sequence of uint16 Frames in, std::vector<RoiMask> bytes
    out, the call compress_sequence makes (pipeline.hpp:142) — on one C3 well, host clock around
    the synchronous call.  The binary is built against the reference headers here (make -C oracle
    dropin) and travels with the snapshot; None when it is absent."""
    exe = os.path.join(ROOT, "oracle", "_ref", "dropin_bench")
    if not os.path.exists(exe):
        return None
    n, h, w = frames.shape
    path = f"/dev/shm/froi_dropin_{os.getpid()}.raw"
    try:
        frames.tofile(path)
        r = subprocess.run([exe, path, str(w), str(h), str(n), str(steps), str(warmup)],
                           capture_output=True, text=True, timeout=600)
    finally:
        if os.path.exists(path):
            os.unlink(path)
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    if r.returncode != 0 or not lines:
        return {"error": (r.stderr or r.stdout)[-300:]}
    d = lines[-1]
    return {"value": d["dropin_frames_per_s"], "unit": UNIT, "ms_per_step": d["ms_per_step"],
            "steps": d["steps"], "frames_per_step": d["frames"],
            "path": "flowroi_gpu::extract_roi(Sequence of uint16 Frames) -> std::vector<RoiMask> "
                    "(pageable host memory both ways; host clock around the call)",
            "masks_match_e2e": (d["mask_pixels"] == ref_pixels) if ref_pixels is not None else None}


# ------------------------------------------------------------------ GPU leg
def run_ours(args) -> None:
    import torch
    from paper_2511_14419_b200 import flowroi, synth
    from paper_2511_14419_b200.params import CFrameStats

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if torch.cuda.device_count() <= local:
        raise SystemExit(f"bench.py: rank {rank} needs cuda:{local}, "
                         f"{torch.cuda.device_count()} device(s) visible")
    numa = bind_numa(local)
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    dist = init_dist(world, "nccl")
    cfg = synth.config("C3")
    F = args.frames
    nsteps = args.warmup + args.steps
    my_wells = wells_for(rank, world, nsteps)
    distinct = sorted(set(my_wells))[: args.distinct_wells]
    # pinned host frames of the distinct wells this rank cycles through
    px = W * H
    host = torch.empty((len(distinct), F, H, W), dtype=torch.uint8, pin_memory=True)
    hv = host.numpy()
    for k, w in enumerate(distinct):
        synth.well_frames(cfg, w, F, out=hv[k])
    slot_of = {w: k for k, w in enumerate(distinct)}
    step_slot = [slot_of.get(w, i % len(distinct)) for i, w in enumerate(my_wells)]
    dev = torch.empty((len(distinct), F, H, W), dtype=torch.uint8, device=device)
    dev.copy_(host)
    SB = (W + 7) // 8
    dmask = torch.empty((F, H, SB), dtype=torch.uint8, device=device)
    hmask = torch.empty((F, H, SB), dtype=torch.uint8, pin_memory=True)
    ctx = flowroi.Context(W, H, 8, cfg.params, device=local, max_pairs=args.max_pairs)
    stream = torch.cuda.ExternalStream(ctx.stream(), device=device)
    torch.cuda.synchronize()

    # ---- device-resident leg
    launches = 0
    kt_sum: dict = {}
    clocks = Clocks(local)
    ev_start, ev_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(args.warmup):
        ctx.extract_wells_device(dev[step_slot[i]].data_ptr(), 1, F, dmask.data_ptr())
    barrier(dist)
    torch.cuda.synchronize()
    clocks.start()
    with torch.cuda.stream(stream):
        ev_start.record(stream)
    for i in range(args.warmup, nsteps):
        ctx.extract_wells_device(dev[step_slot[i]].data_ptr(), 1, F, dmask.data_ptr())
        launches += ctx.launch_count()
    ev_end.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    barrier(dist)
    ms = ev_start.elapsed_time(ev_end)
    # ---- kernel-duration leg: with one execution lane the per-stage events bracket only the
    # stage's own kernels, so they give the kernels' durations for the roofline (the timed leg
    # above overlaps consecutive batches on two lanes)
    ksteps = min(2, args.steps)
    ctx.set_lanes(1)
    ctx.set_fork(False)  # each stage's events bracket only its own kernels
    ctx.extract_wells_device(dev[step_slot[0]].data_ptr(), 1, F, dmask.data_ptr())
    for i in range(args.warmup, args.warmup + ksteps):
        ctx.extract_wells_device(dev[step_slot[i]].data_ptr(), 1, F, dmask.data_ptr())
        for k, v in ctx.kernel_times().items():
            kt_sum[k] = kt_sum.get(k, 0) + v
    ctx.set_lanes(2)
    ctx.set_fork(True)
    torch.cuda.synchronize()
    ms_max = reduce_max(dist, ms, device)
    masks_local = args.steps * F
    masks_all = reduce_sum(dist, float(masks_local), device)
    value = masks_all / (ms_max / 1000.0)

    # ---- end-to-end leg through the public host API
    e2e = None
    if not args.no_e2e:
        stats = (CFrameStats * F)()
        for i in range(min(args.warmup, 2)):
            ctx.extract_wells_into(hv[step_slot[i]][None], hmask.numpy(), stats)
        barrier(dist)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(args.warmup, nsteps):
            ctx.extract_wells_into(hv[step_slot[i]][None], hmask.numpy(), stats)
            _ = hmask[0, 0, 0].item()  # host read of the step's result
        e1.record(stream)
        torch.cuda.synchronize()
        ems = reduce_max(dist, e0.elapsed_time(e1), device)
        e2e = {"value": masks_all / (ems / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": F * px, "d2h_bytes_per_step": F * H * SB + F * 32,
               "ms_per_step": ems / args.steps}

    # ---- the reference-type drop-in (flowroi_gpu::extract_roi over Sequence -> vector<RoiMask>)
    dropin = None
    if rank == 0 and not args.no_dropin:
        last = hv[step_slot[nsteps - 1]]
        ref_pixels = int(np.unpackbits(hmask.numpy()).sum()) if e2e else None
        dropin = run_dropin(last, min(args.steps, 5), 2, ref_pixels)

    # ---- the bit-exact flow mode (froi_ctx_set_flow_exact): same device-resident workload, a few
    # steps; its masks are the reference's byte for byte, so their difference from the fp32 masks
    # of the same well is the default path's end-to-end mismatch rate
    exact = None
    if not args.no_exact:
        ref_fast = dmask.clone()  # fp32-flow masks of the last timed well
        last_slot = step_slot[nsteps - 1]
        ctx.set_flow_exact(True)
        xsteps = min(2, args.steps)
        ctx.extract_wells_device(dev[last_slot].data_ptr(), 1, F, dmask.data_ptr())  # warm-up
        barrier(dist)
        torch.cuda.synchronize()
        x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        x0.record(stream)
        for i in range(xsteps):
            ctx.extract_wells_device(dev[last_slot].data_ptr(), 1, F, dmask.data_ptr())
        x1.record(stream)
        torch.cuda.synchronize()
        xms = reduce_max(dist, x0.elapsed_time(x1), device)
        diff = torch.bitwise_xor(ref_fast, dmask)
        popc = torch.tensor([bin(i).count("1") for i in range(256)], dtype=torch.int64, device=device)
        nd = int(popc[diff.long()].sum().item())
        ctx.set_flow_exact(False)
        exact = {"value": world * xsteps * F / (xms / 1000.0), "unit": UNIT, "steps": xsteps,
                 "ms_per_step": xms / xsteps, "dtype": "f64 flow (bit-exact with the reference)",
                 "fast_path_mask_mismatch": nd / float(F * px),
                 "note": "device-resident, 2 lanes; fp32-path masks of the same well differ from "
                         "these (= the reference's) in fast_path_mask_mismatch of the pixels"}

    # ---- roofline of the fused flow kernel + pipeline figure
    pk = peaks()
    mb = model_bytes_per_pair(W, H, 1, cfg.params.flow.pyramid_levels)
    pairs = kt_sum.get("pairs", 0)
    flow_ns = max(1, kt_sum.get("flow_iter_ns", 1))
    flow_launches = max(1, kt_sum.get("flow_iter_launches", 1))
    achieved = mb["flow"] * pairs / (flow_ns * 1e-9) / 1e9  # GB/s
    roofline = {"bound": "hbm", "kernel": "k_flow_iter", "achieved": achieved,
                "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": achieved / pk["hbm_gbs"],
                "peak_source": pk["source"], "traffic": args.ncu_traffic,
                "bytes_per_launch": mb["flow"] * pairs / flow_launches,
                "avg_launch_us": flow_ns / flow_launches / 1e3,
                "timed_on": f"{ksteps} step(s) with one execution lane and no intra-batch fork (kernel durations)"}
    pairs_per_s = (F - 1) * args.steps / (ms / 1000.0) if ms > 0 else 0.0
    stage_frac = {k.replace("_ns", ""): v / max(1, sum(kt_sum.get(x, 0) for x in (
        "denoise_ns", "fft_forward_ns", "expand_ns", "register_ns", "expand_shifted_ns",
        "flow_iter_ns", "mask_ns"))) for k, v in kt_sum.items() if k.endswith("_ns")}

    # fp64 roofline of the exact-fp64 stages: ncu-counted fp64 instructions per frame / pair
    # (profiles/fp64_work.json) over their event-timed stage time, against the measured fp64 peak
    fp64 = None
    fw = os.path.join(ROOT, "profiles", "fp64_work.json")
    if os.path.exists(fw) and kt_sum.get("pairs"):
        with open(fw) as f:
            w64 = json.load(f)
        pk64 = w64["peak"]["fp64_inst_per_s"]
        fp64 = {"bound": "fp64", "unit": "fp64 inst/s", "peak": pk64, "peak_source": "measured (fp64_peak.cu)"}
        for stage, units, per in (("denoise", kt_sum["frames"], w64["inst_per_frame"]["denoise"]),
                                  ("fft_forward", kt_sum["frames"], w64["inst_per_frame"]["fft_forward"]),
                                  ("register", kt_sum["pairs"], w64["inst_per_pair"]["register"])):
            t = kt_sum.get(stage + "_ns", 0) * 1e-9
            if t > 0:
                ach = per * units / t
                fp64[stage] = {"achieved": ach, "frac": ach / pk64}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        # ~10 s of the reference on every host thread: 8 pairs per thread of one C3 well
        cores = os.cpu_count() or 1
        r = cpu_reference(sample_frames(cores), 0, 1, 0, cores)
        cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "u8 frames; f32 flow; f64 denoise/registration/saliency",
            "data": "synthetic (gen/synth.c seeded C3 wells; ComplexEye data not available)",
            "config": {"workload": "C3: 64 wells x 450 frames, 1024x1024 u8 (one full well per "
                                   "rank per step, well (i*N+r) mod 64)",
                       "frames_per_well": F, "wells_per_step_per_gpu": 1,
                       "global_batch": world * F, "parallelism": f"wells sharded over {world} GPU(s)",
                       "lanes": "2 execution lanes per GPU (consecutive 64-pair batches overlap)",
                       "graphs": "each batch's kernel sequence replayed as a CUDA graph (FROI_GRAPHS=0 disables)",
                       "host": f"one process per GPU; rank 0 NUMA binding: {numa}",
                       "l2": "each step reads a 472 MB well (> 126 MB L2); no flush",
                       "params": "ExtractParams{} defaults (pyramid 3, window 15, threshold 0.2)"},
            "roofline": roofline,
            "pipeline_roofline": {"model_bytes_per_pair": mb["total"],
                                  "achieved_gbs": mb["total"] * pairs_per_s / 1e9,
                                  "frac": mb["total"] * pairs_per_s / 1e9 / pk["hbm_gbs"],
                                  "pairs_per_s_per_gpu": pairs_per_s},
            "stage_share": stage_frac,
            "fp64_roofline": fp64,
            # per-step device time inside the per-stage events of the one-lane leg (vs ms_per_step
            # of the two-lane timed leg)
            "stage_ms_per_step_1lane": sum(kt_sum.get(x, 0) for x in (
                "denoise_ns", "fft_forward_ns", "expand_ns", "register_ns", "expand_shifted_ns",
                "flow_iter_ns", "mask_ns")) / 1e6 / max(1, ksteps),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "dropin_e2e": dropin,
            "exact_flow": exact,
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--frames", type=int, default=450, help="frames per well (C3: 450)")
    ap.add_argument("--distinct-wells", type=int, default=6)
    ap.add_argument("--max-pairs", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dropin", action="store_true")
    ap.add_argument("--no-exact", action="store_true", help="skip the bit-exact flow leg")
    ap.add_argument("--selftest", action="store_true",
                    help="CPU/gloo self-test of the multi-rank launcher (no GPU work)")
    ap.add_argument("--ncu-traffic", type=float, default=None,
                    help="dram bytes per k_flow_iter launch from the committed ncu capture")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.ncu_traffic is None:
        p = os.path.join(ROOT, "profiles", "flow_iter_traffic.json")
        if os.path.exists(p):
            with open(p) as f:
                args.ncu_traffic = json.load(f).get("dram_bytes_per_launch")
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.impl == "reference":
        # the CPU arm runs on rank 0 only; under torchrun the other ranks exit 0 without work
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args.gpus, sys.argv[1:], need_gpus=not args.selftest))
    if args.selftest:
        run_selftest(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
