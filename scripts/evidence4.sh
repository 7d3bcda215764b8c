#!/bin/bash
# Session-4 evidence: bench lines for the resident workloads (engine 6 by
# default) and P3, the launch list of the F bench, one --set full capture of
# the pipelined kernel on F (outputs under gpurun_out/).
mkdir -p gpurun_out
for w in f s csc; do
  timeout 600 python bench.py --workload $w > gpurun_out/e4_bench_$w.json 2> gpurun_out/e4_bench_$w.err
done
timeout 900 python bench.py > gpurun_out/e4_bench_p3.json 2> gpurun_out/e4_bench_p3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/e4_launches_f.csv python bench.py --workload f --steps 2 --warmup 1 --no-cpu-baseline --no-secondary > gpurun_out/e4_ncu_f.log 2>&1
SPCG_CLUS_NONCOOP=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:clus_pcg -c 1 \
  -o gpurun_out/e4_pcg_f python scripts/clus_once.py 0 6 > gpurun_out/e4_ncu_full.log 2>&1
echo done
