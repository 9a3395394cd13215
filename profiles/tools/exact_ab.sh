#!/bin/bash
# exact-flow stage time (one lane, 1 C3 well) for each library variant named on the command line
#   profiles/tools/exact_ab.sh TAG lib1 lib2 ...
TAG=$1; shift
L=paper_2511_14419_b200/_lib
for rep in 1 2; do
  for lib in "$@"; do
    STAGE_AB_EXACT=1 FROI_LIB=$L/$lib timeout 300 python profiles/tools/stage_ab.py $lib 1 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['tag'], 'flow', d['flow_iter_us_per_pair'], 'two_lane', d['two_lane_frames_per_s'], d['mask_checksum'])"
  done
done | tee gpurun_out/${TAG}_ab.log
