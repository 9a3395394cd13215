#!/bin/bash
# usage (on the box): profiles/tools/ncu_one.sh tag "kernel:skip" ...
TAG=$1; shift
python bench.py --steps 1 --warmup 3 --frames 33 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_plain.log 2>&1 || exit 1
for ks in "$@"; do
  k=${ks%%:*}; sk=${ks##*:}
  ncu --set full --clock-control none --import-source on -k regex:"$k" -s $sk -c 1 -o gpurun_out/${TAG}_${k}_$sk python bench.py --steps 1 --warmup 3 --frames 33 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_${k}_$sk.log 2>&1
done
