#!/bin/bash
mkdir -p gpurun_out
CMD="python scripts/solve_once.py P3 0 0"
timeout 300 $CMD > gpurun_out/plain_traffic.log 2>&1 && \
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none -k regex:cg_kernel -c 1 --csv --log-file gpurun_out/traffic_p3.csv $CMD > gpurun_out/ncu_traffic.log 2>&1
echo done
