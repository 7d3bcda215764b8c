#!/bin/bash
# ncu --set full of one pass-A launch (dist_spmv_pq) of a device-generated solve.
# bash scripts/ncu_pq.sh <P3|P2|Q27|Q27P> <tag>
mkdir -p gpurun_out
CMD="python scripts/solve_once.py $1 20 2"
timeout 300 $CMD > gpurun_out/plain_$2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dist_spmv_pq -s 3 -c 1 -o gpurun_out/prof_$2 $CMD > gpurun_out/ncu_$2.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_$2.log
