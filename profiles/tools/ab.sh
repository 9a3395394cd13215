#!/bin/bash
# usage: ab.sh VAR val0 val1  -- alternating A/B bench runs on the box
V=$1; A=$2; B=$3
timeout 300 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "flow or config" 2>&1 | tail -2
for i in 1 2; do for val in $A $B; do
  env $V=$val python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$V=$val', round(d['value'],1), 'flow', round(d['roofline']['avg_launch_us'],1), 'stage1', round(d['stage_ms_per_step_1lane'],2), {k:round(v,3) for k,v in d['stage_share'].items()})"
done; done
