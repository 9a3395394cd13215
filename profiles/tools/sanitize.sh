#!/bin/bash
# compute-sanitizer over the sanitize_cases.py workloads (run on the GPU box via gpurun).
#   profiles/tools/sanitize.sh TAG [case ...]     logs -> gpurun_out/TAG_<tool>_<case>.log
TAG=${1:-r02}; shift
CASES=${@:-c1 lanes u16}
CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out
for c in $CASES; do
  for tool in memcheck racecheck synccheck initcheck; do
    extra=""
    [ "$tool" = memcheck ] && extra="--leak-check full"
    [ "$tool" = racecheck ] && extra="--racecheck-report all"
    timeout 1200 $CS --tool $tool $extra --error-exitcode 9 --print-limit 50 \
      python profiles/tools/sanitize_cases.py $c > gpurun_out/${TAG}_${tool}_${c}.log 2>&1
    echo "$tool $c rc=$?" | tee -a gpurun_out/${TAG}_sanitize_summary.txt
    tail -3 gpurun_out/${TAG}_${tool}_${c}.log
  done
done
