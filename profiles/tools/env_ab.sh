#!/bin/bash
# stage_ab.py (one lane, 3 C3 wells) with and without an environment switch, two rounds.
#   profiles/tools/env_ab.sh TAG VAR        (VAR=0 vs unset)
TAG=$1; VAR=$2
for rep in 1 2; do
  env $VAR=0 timeout 300 python profiles/tools/stage_ab.py "${VAR}=0" 3 | tail -1
  timeout 300 python profiles/tools/stage_ab.py default 3 | tail -1
done | tee gpurun_out/${TAG}_ab.log
