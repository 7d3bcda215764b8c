#!/bin/bash
for k in 1 2 3 8; do
  echo "== K=$k" >> gpurun_out/ncu_k.log
  SPCG_CLUS_K=$k timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:clus_cg python scripts/clus_once.py 0 5 2>&1 | grep -i "RuntimeError\|gpu__time\|^[0-9]" >> gpurun_out/ncu_k.log
  SPCG_CLUS_K=$k timeout 100 python scripts/clus_once.py 0 5 >> gpurun_out/ncu_k.log 2>&1
done
