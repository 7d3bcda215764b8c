#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_generators.py tests/test_gpu_table1.py tests/test_gpu_kernels.py tests/test_gpu_cg.py tests/test_gpu_random_sweep.py tests/test_gpu_c_abi.py -q --timeout 300 -p no:cacheprovider > gpurun_out/check2.log 2>&1; echo pytest_exit=$? >> gpurun_out/check2.log
timeout 900 python bench.py --engine sharded --transport p2p --workload p3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_p2p_p3.log 2>&1; echo bench_p2p=$? >> gpurun_out/bench_p2p_p3.log
timeout 900 python scripts/clus_stress.py 200 6,5,3 > gpurun_out/stress.log 2>&1
tail -5 gpurun_out/check2.log; grep engine gpurun_out/stress.log; tail -c 600 gpurun_out/bench_p2p_p3.log
