#!/bin/bash
# Round-2 ncu evidence (one gpurun call): per-launch DRAM traffic of the
# dominant kernel (dist_spmv_pq) for P3 / P2 / Q27 atomic / Q27 privatized,
# the launch list of the default bench command, and a --set full capture of
# P3's pass A.  Every command ran without ncu first.
mkdir -p gpurun_out/r02
for C in P3 P2 Q27 Q27P; do
  CMD="python scripts/solve_once.py $C 20 2"
  timeout 300 $CMD > gpurun_out/r02/plain_$C.log 2>&1 && \
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum --clock-control none -k regex:dist_spmv_pq -s 3 -c 2 --csv --log-file gpurun_out/r02/traffic_$C.csv $CMD > gpurun_out/r02/ncu_traffic_$C.log 2>&1
done
BENCH="python bench.py --steps 1 --warmup 1 --no-secondary --no-cpu-baseline"
timeout 600 $BENCH > gpurun_out/r02/plain_bench.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02/launches_bench_p3.csv $BENCH > gpurun_out/r02/ncu_bench.log 2>&1
CMD="python scripts/solve_once.py P3 20 2"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dist_spmv_pq -s 3 -c 1 -o gpurun_out/r02/prof_pq_p3 $CMD > gpurun_out/r02/ncu_full_p3.log 2>&1
echo done
ls gpurun_out/r02
