#!/bin/bash
# stage_ab.py (one lane, 3 C3 wells) for each named library build, two interleaved rounds.
#   profiles/tools/ab_stage.sh TAG lib1 lib2 ...      -> gpurun_out/TAG_ab.log
TAG=$1; shift
L=paper_2511_14419_b200/_lib
for rep in 1 2; do
  for lib in "$@"; do
    FROI_LIB=$L/$lib timeout 300 python profiles/tools/stage_ab.py $lib 3 2>&1 | tail -1
  done
done | tee gpurun_out/${TAG}_ab.log
