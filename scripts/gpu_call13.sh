#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --table1 > gpurun_out/table1.json 2> gpurun_out/table1.err
rm -f gpurun_out/variants.log
VARIANTS="cur rowonly" PROBE="Q27F Q27P F" bash scripts/variants.sh
CMD="python bench.py --steps 2 --warmup 1 --max-iter 30 --no-cpu-baseline --no-secondary"
timeout 300 $CMD > gpurun_out/plain_p3.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:cg_kernel -s 1 -c 1 -o gpurun_out/prof_cg_p3_v2 $CMD > gpurun_out/ncu_full_p3.log 2>&1
