import time, threading, torch, numpy as np, sys
sys.path.insert(0, '.')
from paper_2511_14419_b200 import flowroi, ExtractParams
from paper_2511_14419_b200 import synth
F = 450; W = H = 1024
rng = np.random.default_rng(1)
# synthetic C3-like wells via the repo generator
cfg = synth.config("C3")
wells = []
for w in range(4):
    a = synth.well_frames(cfg, w, F)
    wells.append(torch.from_numpy(a).cuda())
torch.cuda.synchronize()
ctxs = [flowroi.Context(W, H, 8, ExtractParams()) for _ in range(2)]
outs = [torch.empty((F, H, (W+7)//8), dtype=torch.uint8, device='cuda') for _ in range(2)]
def run(i, wl, reps):
    for r in range(reps):
        for w in wl:
            ctxs[i].extract_wells_device(wells[w].data_ptr(), 1, F, outs[i].data_ptr())
for i in range(2): run(i, [0], 1)
torch.cuda.synchronize()
t = time.perf_counter(); run(0, [0,1,2,3], 1); torch.cuda.synchronize(); t1 = time.perf_counter()-t
print('one ctx: 4 wells', t1*1e3, 'ms ->', 4*F/t1, 'frames/s')
t = time.perf_counter()
th = [threading.Thread(target=run, args=(0,[0,1],1)), threading.Thread(target=run, args=(1,[2,3],1))]
[x.start() for x in th]; [x.join() for x in th]; torch.cuda.synchronize(); t2 = time.perf_counter()-t
print('two ctx threads: 4 wells', t2*1e3, 'ms ->', 4*F/t2, 'frames/s')
