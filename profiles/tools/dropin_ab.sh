#!/bin/bash
# drop-in end to end (oracle/_ref/dropin_bench, one C3 well x 450) for each named library build
python - "$@" <<'PY'
import os, subprocess, sys
sys.path.insert(0, ".")
from paper_2511_14419_b200 import synth
fr = synth.well_frames(synth.config("C3"), 0, 450)
fr.tofile("/dev/shm/froi_dropin_ab.raw")
L = "paper_2511_14419_b200/_lib"
for rep in range(2):
    for lib in sys.argv[1:]:
        # the binary's rpath points at _lib/libfroi.so: preload the build under test
        env = dict(os.environ, LD_PRELOAD=os.path.abspath(os.path.join(L, lib)))
        r = subprocess.run(["oracle/_ref/dropin_bench", "/dev/shm/froi_dropin_ab.raw", "1024", "1024", "450", "5", "2"],
                           capture_output=True, text=True, env=env)
        print(lib, r.stdout.strip()[-160:], r.stderr[-200:], flush=True)
os.unlink("/dev/shm/froi_dropin_ab.raw")
PY
