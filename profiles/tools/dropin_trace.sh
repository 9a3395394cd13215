python - <<'PY'
import os, subprocess, sys
sys.path.insert(0, ".")
from paper_2511_14419_b200 import synth
fr = synth.well_frames(synth.config("C3"), 0, 450)
fr.tofile("/dev/shm/froi_dt.raw")
print("cpus", os.cpu_count(), flush=True)
env = dict(os.environ, FROI_TRACE="1")
r = subprocess.run(["oracle/_ref/dropin_bench", "/dev/shm/froi_dt.raw", "1024", "1024", "450", "3", "2"], capture_output=True, text=True, env=env)
print(r.stdout[-400:]); print(r.stderr[-6000:])
PY
lscpu | head -20; free -g
