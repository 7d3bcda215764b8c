#!/bin/bash
mkdir -p gpurun_out
CMD="python scripts/clus_once.py 0 5"
timeout 300 $CMD > gpurun_out/plain_clus.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:clus_cg -s 1 -c 1 -o gpurun_out/prof_clus $CMD > gpurun_out/ncu_clus.log 2>&1
echo done
