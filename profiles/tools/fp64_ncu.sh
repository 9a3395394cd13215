#!/bin/bash
# fp64 work of the exact-fp64 kernels (denoise, registration FFTs, mask-stage producer), for their
# fp64 roofline: executed DADD/DMUL/DFMA thread instructions and duration per launch.
#   profiles/tools/fp64_ncu.sh TAG     -> gpurun_out/TAG_fp64.csv
TAG=${1:-r02}
M=gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:"k_denoise|k_fft|k_xpow|k_inv_cols|k_argmax|k_mag_grad" \
  -c 24 --csv --log-file gpurun_out/${TAG}_fp64.csv python profiles/tools/stage_ab.py ncu 1 > gpurun_out/${TAG}_fp64.out 2>&1
echo "fp64 ncu rc=$?"
