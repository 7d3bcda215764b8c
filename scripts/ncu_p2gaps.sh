#!/bin/bash
CMD="python scripts/solve_once.py P2 40 2"
timeout 300 $CMD > gpurun_out/plain_p2.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_p2.csv $CMD > gpurun_out/ncu_p2.log 2>&1
echo done
