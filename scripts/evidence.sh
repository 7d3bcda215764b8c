#!/bin/bash
# Bench lines for every workload + the ncu launch list of the default bench
# command (one gpurun call; outputs under gpurun_out/).
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/ev_bench_p3.json 2> gpurun_out/ev_bench_p3.err
for w in p2 q27 q27p f s csc; do
  timeout 600 python bench.py --workload $w > gpurun_out/ev_bench_$w.json 2> gpurun_out/ev_bench_$w.err
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev_bench_ref.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/ev_launches_p3.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ev_ncu_bench.log 2>&1
echo done
