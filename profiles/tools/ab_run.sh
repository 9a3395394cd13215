#!/bin/bash
# A/B on the GPU box: stage_ab.py with each library build named on the command line, twice each
# interleaved, then the bench e2e leg with each.   profiles/tools/ab_run.sh TAG lib1 lib2 ...
TAG=$1; shift
L=paper_2511_14419_b200/_lib
for rep in 1 2; do
  for lib in "$@"; do
    FROI_LIB=$L/$lib timeout 300 python profiles/tools/stage_ab.py $lib 3 2>&1 | tail -1
  done
done | tee gpurun_out/${TAG}_ab.log
if [ -n "$AB_E2E" ]; then
  for lib in "$@"; do
    FROI_LIB=$L/$lib timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-dropin 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
  done | tee -a gpurun_out/${TAG}_ab.log
fi
