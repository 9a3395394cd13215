"""Multi-rank host logic on CPU (gloo, world_size 2): well sharding and the max/sum reductions the
bench uses for its whole-job throughput (no GPU, no data-path collective)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch
    import torch.distributed as dist

    import bench
    r, w, l = bench.dist_env()
    d = bench.init_dist(w, "gloo")
    wells = bench.wells_for(r, w, 8)
    # per-rank device time and mask counts, reduced like the bench does
    t = bench.reduce_max(d, 100.0 + 10 * r, torch.device("cpu"))
    n = bench.reduce_sum(d, float(len(wells) * 450), torch.device("cpu"))
    bench.barrier(d)
    q.put((r, wells, t, n))
    dist.destroy_process_group()


def test_two_rank_sharding_and_reductions():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, w0, t0, n0), (r1, w1, t1, n1) = out
    assert set(w0).isdisjoint(w1)                       # wells never split across ranks
    assert all(w % 2 == 0 for w in w0) and all(w % 2 == 1 for w in w1)
    assert t0 == t1 == 110.0                            # max over ranks
    assert n0 == n1 == 2 * 8 * 450                      # whole-job frame count


def test_shard_wells_assignment():
    from paper_2511_14419_b200.flowroi import shard_wells
    s = shard_wells(64, [0, 1, 2, 3, 4, 5, 6, 7])
    assert sorted(w for ws in s.values() for w in ws) == list(range(64))
    assert all(len(ws) == 8 for ws in s.values())
    assert s[3] == [3, 11, 19, 27, 35, 43, 51, 59]


def _bench(*args, timeout=180):
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                          capture_output=True, text=True, timeout=timeout, env=env)


def test_bench_launcher_spawns_n_ranks():
    """`bench.py --gpus 2` with no external launcher spawns two ranks (gloo self-test mode):
    rank 0 prints one line with n_gpus 2, the max over ranks and the whole-job frame count."""
    import json
    r = _bench("--gpus", "2", "--selftest", "--steps", "4", "--warmup", "3")
    assert r.returncode == 0, r.stderr
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = lines[0]
    assert d["n_gpus"] == 2 and d["ms_max"] == 110.0
    assert d["frames"] == 2 * 4 * 450
    w0, w1 = d["wells"]
    assert w0 == [6, 8, 10, 12] and w1 == [7, 9, 11, 13]


def test_bench_refuses_missing_gpus():
    """Asking for more GPUs than are visible fails loudly instead of measuring fewer."""
    import torch
    n = torch.cuda.device_count() + 1
    r = _bench("--gpus", str(n), "--steps", "1", "--warmup", "3", timeout=120)
    assert r.returncode != 0
    assert "visible" in r.stderr
