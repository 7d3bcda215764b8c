#!/bin/bash
# Session-4 evidence (outputs under gpurun_out/): engine 5 vs 6 per-solve
# distribution, the GPU suite + smoke, bench lines for the resident workloads
# (engine 6 by default), the launch list of the F bench and one --set full
# capture of the pipelined kernel on F.  SPCG_CLUS_NONCOOP=1 under ncu: ncu
# drops the cluster shape of a cooperative cluster launch.
mkdir -p gpurun_out
timeout 300 python scripts/pipe_dist.py 15 5,6 > gpurun_out/e4_dist.log 2>&1
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/e4_pytest.log 2>&1; echo pytest_exit=$? >> gpurun_out/e4_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/e4_pytest.log 2>&1
for w in f s csc; do
  timeout 600 python bench.py --workload $w > gpurun_out/e4_bench_$w.json 2> gpurun_out/e4_bench_$w.err
done
SPCG_CLUS_NONCOOP=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/e4_launches_f.csv python bench.py --workload f --steps 2 --warmup 1 --no-cpu-baseline --no-secondary > gpurun_out/e4_ncu_f.log 2>&1
SPCG_CLUS_NONCOOP=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:clus_pcg -c 1 \
  -o gpurun_out/e4_pcg_f2 python scripts/clus_once.py 0 6 > gpurun_out/e4_ncu_full.log 2>&1
echo done
