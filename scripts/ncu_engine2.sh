#!/bin/bash
mkdir -p gpurun_out
CMD="python scripts/solve_once.py P3 30 2"
timeout 300 $CMD > gpurun_out/plain_e2.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_e2.csv $CMD > gpurun_out/ncu_e2.log 2>&1
echo done
