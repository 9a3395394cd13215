#!/bin/bash
# on the box: default bench, then the ncu launch list (first 600 launches) and one full capture of
# a level-0 k_flow_iter launch, same bench command (CPU-baseline leg off under ncu: no kernels)
T=$1
python bench.py > gpurun_out/${T}_bench.log 2>&1 || { tail -5 gpurun_out/${T}_bench.log; exit 1; }
tail -1 gpurun_out/${T}_bench.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --no-cpu-baseline > gpurun_out/${T}_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_flow_iter -s 6 -c 1 -o gpurun_out/${T}_flow python bench.py --no-cpu-baseline > gpurun_out/${T}_ncu2.log 2>&1
ls -la gpurun_out | grep $T
