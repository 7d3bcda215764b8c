#!/bin/bash
mkdir -p gpurun_out
CMD="python scripts/clus_once.py 0 5"
for mode in "--replay-mode application" "--replay-mode kernel" "--cache-control none" "--launch-skip 0 --launch-count 1 --replay-mode application"; do
  echo "== $mode" >> gpurun_out/ncu_modes.log
  timeout 300 ncu $mode --metrics gpu__time_duration.sum --clock-control none -k regex:clus_cg $CMD >> gpurun_out/ncu_modes.log 2>&1
  echo "exit=$?" >> gpurun_out/ncu_modes.log
done
echo "== no ncu, CUDA_LAUNCH_BLOCKING=1" >> gpurun_out/ncu_modes.log
CUDA_LAUNCH_BLOCKING=1 timeout 120 $CMD >> gpurun_out/ncu_modes.log 2>&1
