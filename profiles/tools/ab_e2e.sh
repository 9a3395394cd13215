#!/bin/bash
# usage (on the box): profiles/tools/ab_e2e.sh VAR v1 v2 ... -- alternating default benches
# (device + end-to-end legs, no CPU leg), one per value of the environment variable VAR
V=$1; shift
for i in 1 2; do for val in "$@"; do
  env $V=$val python bench.py --steps 6 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$V=$val', 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'launches', d['gpu_launches'])"
done; done
