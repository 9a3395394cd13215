"""Where the end-to-end leg loses time against the device leg (450-frame 1024^2 well):
device call, host call, and the bare H2D / D2H copies, CUDA-event timed on the context stream."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_14419_b200 import flowroi, ExtractParams
from paper_2511_14419_b200.params import CFrameStats
from paper_2511_14419_b200 import synth

F, W, H = 450, 1024, 1024
frames = synth.well_frames(synth.config("C3"), 0, F)
hv = torch.empty((F, H, W), dtype=torch.uint8, pin_memory=True)
hv.numpy()[:] = frames
dv = hv.cuda()
hm = torch.empty((F, H, (W + 7) // 8), dtype=torch.uint8, pin_memory=True)
dm = torch.empty_like(hm, device='cuda')
ctx = flowroi.Context(W, H, 8, ExtractParams())
stream = torch.cuda.ExternalStream(ctx.stream())
stats = (CFrameStats * F)()

def timed(fn, n=3):
    out = []
    for _ in range(n):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = time.perf_counter()
        e0.record(stream); fn(); e1.record(stream)
        torch.cuda.synchronize()
        out.append((e0.elapsed_time(e1), (time.perf_counter() - t) * 1e3))
    return out

print('H2D copy', timed(lambda: dv.copy_(hv, non_blocking=True)))
print('D2H copy', timed(lambda: hm.copy_(dm, non_blocking=True)))
print('device call', timed(lambda: ctx.extract_wells_device(dv.data_ptr(), 1, F, dm.data_ptr())))
print('host call', timed(lambda: ctx.extract_wells_into(hv.numpy()[None], hm.numpy(), stats)))
ctx.set_lanes(1)
print('device call 1 lane', timed(lambda: ctx.extract_wells_device(dv.data_ptr(), 1, F, dm.data_ptr())))
print('host call 1 lane', timed(lambda: ctx.extract_wells_into(hv.numpy()[None], hm.numpy(), stats)))

# contention probe: the device call while the copy engine uploads a well on another stream
ctx.set_lanes(2)
side = torch.cuda.Stream()
dv2 = torch.empty_like(dv)
def dev_with_copy():
    with torch.cuda.stream(side):
        dv2.copy_(hv, non_blocking=True)
    ctx.extract_wells_device(dv.data_ptr(), 1, F, dm.data_ptr())
print('device call + concurrent H2D', timed(dev_with_copy))
# host call with a pageable mask destination (no per-batch read-back; one copy at the end)
hm_pageable = np.empty(hm.shape, dtype=np.uint8)
print('host call, pageable masks', timed(lambda: ctx.extract_wells_into(hv.numpy()[None], hm_pageable, stats)))
