#!/bin/bash
# drop-in end-to-end (oracle/_ref/dropin_bench on one C3 well) for several host-thread counts
python - <<'PY'
import os, subprocess, sys, json
sys.path.insert(0, ".")
from paper_2511_14419_b200 import synth
fr = synth.well_frames(synth.config("C3"), 0, 450)
fr.tofile("/dev/shm/froi_dropin_threads.raw")
print("cpus", os.cpu_count(), flush=True)
for t in ("4", "8", "12", "14", "16"):
    env = dict(os.environ, FROI_HOST_THREADS=t)
    r = subprocess.run(["oracle/_ref/dropin_bench", "/dev/shm/froi_dropin_threads.raw", "1024", "1024", "450", "5", "2"],
                       capture_output=True, text=True, env=env)
    print("threads", t, r.stdout.strip()[-200:], r.stderr[-200:], flush=True)
os.unlink("/dev/shm/froi_dropin_threads.raw")
PY
