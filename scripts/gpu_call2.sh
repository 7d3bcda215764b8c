#!/bin/bash
# bench + ncu evidence (run under gpurun from the repo root)
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench_exit=$? >> gpurun_out/bench.err
timeout 300 python scripts/probe.py P2 Q27 Q27P > gpurun_out/probe2.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --max-iter 30 --no-cpu-baseline --no-secondary"
timeout 300 $CMD > gpurun_out/plain_p3.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_p3.csv $CMD > gpurun_out/ncu_launch.log 2>&1
timeout 300 $CMD > gpurun_out/plain_p3b.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:cg_kernel -s 1 -c 1 -o gpurun_out/prof_cg_p3 $CMD > gpurun_out/ncu_full_p3.log 2>&1
CMDF="python bench.py --workload f --steps 2 --warmup 1 --no-cpu-baseline --no-secondary"
timeout 300 $CMDF > gpurun_out/plain_f.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:cg_kernel -s 1 -c 1 -o gpurun_out/prof_cg_f $CMDF > gpurun_out/ncu_full_f.log 2>&1
echo done
