#!/bin/bash
# k_flow_iter at one CTA per SM (leaving registers / shared memory for the other lane's kernels)
# vs two: one-lane stage times and two-lane bench value.   profiles/tools/flow_1cta_ab.sh TAG
TAG=$1
L=paper_2511_14419_b200/_lib
run_bench() {  # label, env...
  local lab=$1; shift
  env "$@" timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-dropin 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lab', 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'flow_us', round(d['roofline']['avg_launch_us'],1))"
}
for rep in 1 2; do
  timeout 300 python profiles/tools/stage_ab.py default 3 | tail -1
  FROI_FLOW_SMEM_MIN=120000 timeout 300 python profiles/tools/stage_ab.py smem120k 3 | tail -1
  FROI_LIB=$L/libfroi_fm1.so timeout 300 python profiles/tools/stage_ab.py minb1 3 | tail -1
  run_bench default FROI_X=0
  run_bench smem120k FROI_FLOW_SMEM_MIN=120000
  run_bench minb1 FROI_LIB=$L/libfroi_fm1.so
done 2>&1 | tee gpurun_out/${TAG}_ab.log
