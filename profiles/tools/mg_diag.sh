#!/bin/bash
# k_mag_grad duration (ncu, 6 launches of one C3 well) for each named library build
for lib in "$@"; do
  FROI_LIB=paper_2511_14419_b200/_lib/$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_mag_grad -c 6 --csv python profiles/tools/stage_ab.py $lib 1 2>/dev/null | grep gpu__time | awk -F'","' -v L=$lib '{gsub(/"/,"",$NF); s+=$NF; n++} END {print L, n, s/n/1000, "us"}'
done
