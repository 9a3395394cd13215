#!/bin/bash
for nr in 1 2 4 8; do
  FROI_NR=$nr python bench.py --steps 3 --warmup 3 --frames 64 --no-cpu-baseline --no-e2e > gpurun_out/nr$nr.log 2>&1
  echo nr=$nr $(tail -1 gpurun_out/nr$nr.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['roofline']['avg_launch_us'])")
done
