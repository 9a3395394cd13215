"""Per-stage device time of the C3 workload for A/B experiments (run on the GPU box).

  FROI_LIB=paper_2511_14419_b200/_lib/libfroi_base.so python profiles/tools/stage_ab.py TAG [wells]

STAGE_AB_EXACT=1 times the bit-exact fp64 flow mode.  Runs `wells` full C3 wells (450 frames, device-resident) with ONE execution lane, so each stage's
events bracket only its own kernels, and prints one JSON line: us per pair per stage, the flow
kernel's launch count/average, and the two-lane frames/s of the same wells.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2511_14419_b200 import flowroi, synth  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "run"
nw = int(sys.argv[2]) if len(sys.argv) > 2 else 3
max_pairs = int(sys.argv[3]) if len(sys.argv) > 3 else 0
# STAGE_AB_CONFIG=C4 (or C2): the same measurement on another BASELINE configuration
cfg = synth.config(os.environ.get("STAGE_AB_CONFIG", "C3"))
F, W, H = cfg.n_frames, cfg.width, cfg.height
u16 = cfg.sample_bytes == 2
frames = torch.empty((nw, F, H, W), dtype=torch.int16 if u16 else torch.uint8)
for w in range(nw):
    synth.well_frames(cfg, w, F, out=frames[w].numpy().view("uint16" if u16 else "uint8"))
dev = frames.cuda()
masks = torch.empty((F, H, (W + 7) // 8), dtype=torch.uint8, device="cuda")
ctx = flowroi.Context(W, H, cfg.depth, cfg.params, max_pairs=max_pairs)
ctx.set_lanes(1)
if os.environ.get("STAGE_AB_NOFORK"):
    ctx.set_fork(False)
if os.environ.get("STAGE_AB_EXACT"):  # the bit-exact fp64 flow
    ctx.set_flow_exact(True)
ctx.extract_wells_device(dev[0].data_ptr(), 1, F, masks.data_ptr())  # warm-up
acc = {}
for w in range(nw):
    ctx.extract_wells_device(dev[w].data_ptr(), 1, F, masks.data_ptr())
    for k, v in ctx.kernel_times().items():
        acc[k] = acc.get(k, 0) + v
pairs = acc["pairs"]
out = {"tag": tag, "lib": os.environ.get("FROI_LIB", "default")}
for k, v in acc.items():
    if k.endswith("_ns"):
        out[k.replace("_ns", "_us_per_pair")] = round(v / 1e3 / pairs, 3)
out["flow_iter_avg_launch_us"] = round(acc["flow_iter_ns"] / 1e3 / acc["flow_iter_launches"], 2)
out["stage_us_per_pair"] = round(sum(v for k, v in acc.items() if k.endswith("_ns")) / 1e3 / pairs, 2)
ctx.set_lanes(2)
ctx.set_fork(True)
ctx.extract_wells_device(dev[0].data_ptr(), 1, F, masks.data_ptr())
s = torch.cuda.ExternalStream(ctx.stream())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(s)
for w in range(nw):
    ctx.extract_wells_device(dev[w].data_ptr(), 1, F, masks.data_ptr())
e1.record(s)
torch.cuda.synchronize()
out["two_lane_frames_per_s"] = round(nw * F / (e0.elapsed_time(e1) / 1e3), 1)
out["mask_checksum"] = int(masks.to(torch.int64).sum().item())
print(json.dumps(out), flush=True)
ctx.close()
