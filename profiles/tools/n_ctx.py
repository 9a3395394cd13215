import time, threading, torch, numpy as np, sys
sys.path.insert(0, '.')
from paper_2511_14419_b200 import flowroi, ExtractParams, synth
F = 450; W = H = 1024
cfg = synth.config("C3")
wells = [torch.from_numpy(synth.well_frames(cfg, w, F)).cuda() for w in range(6)]
torch.cuda.synchronize()
ctxs = [flowroi.Context(W, H, 8, ExtractParams()) for _ in range(3)]
for c in ctxs: c.set_lanes(1)
outs = [torch.empty((F, H, (W+7)//8), dtype=torch.uint8, device='cuda') for _ in range(3)]
def run(i, wl):
    for w in wl:
        ctxs[i].extract_wells_device(wells[w].data_ptr(), 1, F, outs[i].data_ptr())
for i in range(3): run(i, [0])
torch.cuda.synchronize()
for n in (1, 2, 3):
    parts = [list(range(6))[i::n] for i in range(n)]
    t = time.perf_counter()
    th = [threading.Thread(target=run, args=(i, parts[i])) for i in range(n)]
    [x.start() for x in th]; [x.join() for x in th]; torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(n, 'contexts: 6 wells', round(dt*1e3,1), 'ms ->', round(6*F/dt,1), 'frames/s')
ctxs[0].set_lanes(2)
t = time.perf_counter(); run(0, list(range(6))); torch.cuda.synchronize(); dt = time.perf_counter()-t
print('1 context, 2 lanes: 6 wells', round(dt*1e3,1), 'ms ->', round(6*F/dt,1))
