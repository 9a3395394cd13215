#!/bin/bash
# usage (on the box): profiles/tools/ncu_multi.sh tag kernel1 kernel2 ...
TAG=$1; shift
python bench.py --steps 1 --warmup 3 --frames 33 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_plain.log 2>&1 || exit 1
for k in "$@"; do
  ncu --set full --clock-control none --import-source on -k regex:"$k" -s 2 -c 1 -o gpurun_out/${TAG}_$k python bench.py --steps 1 --warmup 3 --frames 33 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_$k.log 2>&1
done
ls gpurun_out
