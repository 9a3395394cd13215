#!/bin/bash
# drop-in end-to-end with and without glibc malloc tunables that keep 1 MB RoiMask buffers off mmap
python - <<'PY'
import os, subprocess, sys
sys.path.insert(0, ".")
from paper_2511_14419_b200 import synth
fr = synth.well_frames(synth.config("C3"), 0, 450)
fr.tofile("/dev/shm/froi_dm.raw")
for tun in ("", "glibc.malloc.mmap_threshold=33554432:glibc.malloc.trim_threshold=1073741824", "glibc.malloc.arena_max=1"):
    env = dict(os.environ, FROI_TRACE="1")
    if tun: env["GLIBC_TUNABLES"] = tun
    r = subprocess.run(["oracle/_ref/dropin_bench", "/dev/shm/froi_dm.raw", "1024", "1024", "450", "5", "2"], capture_output=True, text=True, env=env)
    print("tunables:", tun or "(none)", r.stdout.strip()[-160:], flush=True)
    print("\n".join(r.stderr.strip().splitlines()[-2:]), flush=True)
os.unlink("/dev/shm/froi_dm.raw")
PY
