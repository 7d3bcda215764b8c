#!/bin/bash
mkdir -p gpurun_out
CMD="python scripts/clus_once.py 0 5"
timeout 300 $CMD > gpurun_out/plain_clus3.log 2>&1 && \
SPCG_CLUS_NONCOOP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:clus_cg -s 1 -c 1 -o gpurun_out/prof_clus_k15 $CMD > gpurun_out/ncu_clus3.log 2>&1
CMD2="python bench.py --workload f --steps 2 --warmup 1 --no-cpu-baseline --no-secondary"
timeout 300 $CMD2 > gpurun_out/plain_benchf.log 2>&1 && \
SPCG_CLUS_NONCOOP=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file gpurun_out/launches_f.csv $CMD2 > gpurun_out/ncu_benchf.log 2>&1
echo done
