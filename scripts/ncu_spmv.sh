#!/bin/bash
mkdir -p gpurun_out
CMD="python scripts/spmv_once.py Q27F 3"
timeout 300 $CMD > gpurun_out/plain_spmv.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_kernel -s 2 -c 1 -o gpurun_out/prof_spmv_q27f $CMD > gpurun_out/ncu_spmv.log 2>&1
CMD2="python scripts/spmv_once.py P3 3"
timeout 300 $CMD2 > gpurun_out/plain_spmv2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_kernel -s 2 -c 1 -o gpurun_out/prof_spmv_p3 $CMD2 > gpurun_out/ncu_spmv2.log 2>&1
echo done
