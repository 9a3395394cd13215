#!/bin/bash
# usage (on the box): profiles/tools/ab.sh VAR v1 v2 ... -- flow/config parity tests, then two
# alternating rounds of short benches, one per value of the environment variable VAR
V=$1; shift
timeout 300 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "flow or config or extract" 2>&1 | tail -2
for i in 1 2; do for val in "$@"; do
  env $V=$val python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$V=$val', round(d['value'],1), 'flow', round(d['roofline']['avg_launch_us'],1), 'stage1', round(d['stage_ms_per_step_1lane'],2), {k:round(v,3) for k,v in d['stage_share'].items()})"
done; done
