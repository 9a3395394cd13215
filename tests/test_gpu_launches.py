"""The launch count the bench reports (`gpu_launches`, from `froi_ctx_launch_count`) is checked
against the kernels CUPTI actually sees for the same call (torch.profiler's CUDA activity), on
both the device-resident and the host (end-to-end) entry points, and every traced kernel is one
of this library's own (no library or fallback kernels on the path)."""
import numpy as np
import pytest

from fixtures import textured_frame

pytestmark = pytest.mark.gpu


def _traced_kernels(fn):
    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type.name == "CUDA" and "memcpy" not in e.name.lower()
             and "memset" not in e.name.lower()]
    return names


@pytest.mark.parametrize("host", [False, True])
def test_launch_count_matches_trace(host):
    import torch
    from paper_2511_14419_b200 import flowroi
    from paper_2511_14419_b200.params import ExtractParams
    W = H = 256
    n = 40  # two batches of up to 32 pairs
    frames = np.stack([textured_frame(W, H, 8, 900 + t) for t in range(n)]).astype(np.uint8)
    ctx = flowroi.Context(W, H, 8, ExtractParams(), device=0, max_pairs=32)
    try:
        if host:
            out = np.zeros((n, H, (W + 7) // 8), np.uint8)
            call = lambda: ctx.extract_wells_into(frames[None], out[None])
        else:
            d = torch.from_numpy(frames).cuda()
            dm = torch.zeros((n, H, (W + 7) // 8), dtype=torch.uint8, device="cuda")
            call = lambda: ctx.extract_wells_device(d.data_ptr(), 1, n, dm.data_ptr())
        call()  # warm-up (lazy allocations, second lane)
        names = _traced_kernels(call)
        if not names:
            pytest.skip("CUPTI kernel activity unavailable in this torch build")
        count = ctx.launch_count()
    finally:
        ctx.close()
    assert all(k.split("(")[0].split("<")[0].split("::")[-1].startswith("k_") or "froi" in k
               for k in names), sorted(set(names))
    assert count == len(names), (count, len(names))
