#!/bin/bash
# usage (on the box): profiles/tools/launch_list.sh TAG [bench args] -- ncu launch list of a short run
T=$1; shift
python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/${T}_plain.log 2>&1 || { tail -5 gpurun_out/${T}_plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/${T}_ncu.log 2>&1
ls -la gpurun_out | grep ${T}
