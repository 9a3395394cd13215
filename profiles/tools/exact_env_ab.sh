#!/bin/bash
# exact-flow stage time (one lane, 1 C3 well) with and without an environment switch, two rounds
#   profiles/tools/exact_env_ab.sh TAG VAR   (VAR=0 vs unset)
TAG=$1; VAR=$2
for rep in 1 2; do
  for lab in "$VAR=0" default; do
    if [ "$lab" = default ]; then E=""; else E="$lab"; fi
    env $E STAGE_AB_EXACT=1 timeout 300 python profiles/tools/stage_ab.py "$lab" 1 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['tag'], 'flow', d['flow_iter_us_per_pair'], 'two_lane', d['two_lane_frames_per_s'], d['mask_checksum'])"
  done
done | tee gpurun_out/${TAG}_ab.log
