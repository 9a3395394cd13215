#!/bin/bash
# forward FFT in L2-sized frame groups (FROI_FFT_GROUP) vs one group: one-lane stage times and
# the two-lane frames/s of stage_ab.py, then the bench value.   profiles/tools/fftgroup_ab.sh TAG
TAG=$1
for rep in 1 2; do
  for G in 0 4 6; do
    FROI_FFT_GROUP=$G timeout 300 python profiles/tools/stage_ab.py G$G 3 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['tag'], 'fft', d['fft_forward_us_per_pair'], 'stage', d['stage_us_per_pair'], 'two_lane', d['two_lane_frames_per_s'], d['mask_checksum'])"
  done
done 2>&1 | tee gpurun_out/${TAG}_ab.log
for G in 0 6; do
  FROI_FFT_GROUP=$G timeout 300 python bench.py --no-cpu-baseline --no-dropin --no-exact 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench G$G', 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
done 2>&1 | tee -a gpurun_out/${TAG}_ab.log
