#!/bin/bash
mkdir -p gpurun_out
CMD="python scripts/spmv_once.py Q27 3"
timeout 300 $CMD > gpurun_out/plain_q27.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_kernel -s 2 -c 1 -o gpurun_out/prof_spmv_q27b $CMD > gpurun_out/ncu_q27.log 2>&1
CMD="python scripts/solve_once.py Q27 20 2"
timeout 300 $CMD > gpurun_out/plain_q27s.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dist_spmv_pq -s 3 -c 1 -o gpurun_out/prof_pq_q27b $CMD > gpurun_out/ncu_q27s.log 2>&1
echo done
