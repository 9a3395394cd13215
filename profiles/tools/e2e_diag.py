import time, torch, numpy as np, sys
sys.path.insert(0, '.')
from paper_2511_14419_b200 import flowroi, ExtractParams
from paper_2511_14419_b200 import synth
F = 450
W = H = 1024
hv = torch.empty((F, H, W), dtype=torch.uint8, pin_memory=True)
cfg = synth.config("C3") if hasattr(synth, "config") else None
frames = np.random.default_rng(1).integers(0, 255, (F, H, W), dtype=np.uint8)
hv.numpy()[:] = frames
dv = torch.empty((F, H, W), dtype=torch.uint8, device='cuda')
torch.cuda.synchronize()
for _ in range(2):
    t = time.perf_counter(); dv.copy_(hv, non_blocking=True); torch.cuda.synchronize(); print('H2D 472MB ms', (time.perf_counter()-t)*1e3)
hm = torch.empty((F, H, (W+7)//8), dtype=torch.uint8, pin_memory=True)
dm = torch.empty_like(hm, device='cuda')
for _ in range(2):
    t = time.perf_counter(); hm.copy_(dm, non_blocking=True); torch.cuda.synchronize(); print('D2H masks ms', (time.perf_counter()-t)*1e3)
ctx = flowroi.Context(W, H, 8, ExtractParams())
from paper_2511_14419_b200.params import CFrameStats
stats = (CFrameStats * F)()
for i in range(3):
    t = time.perf_counter(); ctx.extract_wells_into(hv.numpy()[None], hm.numpy(), stats); print('e2e call ms', (time.perf_counter()-t)*1e3)
for i in range(3):
    t = time.perf_counter(); ctx.extract_wells_device(dv.data_ptr(), 1, F, dm.data_ptr()); torch.cuda.synchronize(); print('device call ms', (time.perf_counter()-t)*1e3)
