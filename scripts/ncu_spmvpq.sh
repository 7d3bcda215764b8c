#!/bin/bash
mkdir -p gpurun_out
CMD="python scripts/solve_once.py P3 20 2"
timeout 300 $CMD > gpurun_out/plain_pq.log 2>&1 && \
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none -k regex:dist_spmv_pq -s 3 -c 1 --csv --log-file gpurun_out/traffic_pq.csv $CMD > gpurun_out/ncu_pq.log 2>&1
timeout 300 $CMD > gpurun_out/plain_pq2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dist_spmv_pq -s 3 -c 1 -o gpurun_out/prof_pq $CMD > gpurun_out/ncu_pq_full.log 2>&1
timeout 300 $CMD > gpurun_out/plain_pq3.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_engine2.csv $CMD > gpurun_out/ncu_launch2.log 2>&1
echo done
