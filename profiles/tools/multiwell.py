import os, sys, json, torch
sys.path.insert(0, ".")
from paper_2511_14419_b200 import flowroi, synth
cfg = synth.config("C3"); F = 450; nw = 3
frames = torch.empty((nw, F, 1024, 1024), dtype=torch.uint8)
for w in range(nw): synth.well_frames(cfg, w, F, out=frames[w].numpy())
dev = frames.cuda()
masks = torch.empty((nw * F, 1024, 128), dtype=torch.uint8, device="cuda")
ctx = flowroi.Context(1024, 1024, 8, cfg.params)
s = torch.cuda.ExternalStream(ctx.stream())
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = []
    for _ in range(reps):
        e0.record(s); fn(); e1.record(s); torch.cuda.synchronize(); best.append(e0.elapsed_time(e1))
    return min(best)
sep = t(lambda: [ctx.extract_wells_device(dev[w].data_ptr(), 1, F, masks.data_ptr()) for w in range(nw)])
one = t(lambda: ctx.extract_wells_device(dev.data_ptr(), nw, F, masks.data_ptr()))
print(json.dumps({"separate_ms": sep, "one_call_ms": one, "sep_fps": nw*F/sep*1e3, "one_fps": nw*F/one*1e3}))
