#!/bin/bash
mkdir -p gpurun_out
CMD="python scripts/spmv_once.py Q27F 3"
timeout 300 $CMD > gpurun_out/plain_q27f.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_kernel -s 2 -c 1 -o gpurun_out/prof_spmv_q27f_split $CMD > gpurun_out/ncu_q27f.log 2>&1
echo done
