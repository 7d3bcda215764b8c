#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_dist.py tests/test_gpu_multirank.py tests/test_gpu_cg.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/p2p.log 2>&1; echo pytest_exit=$? >> gpurun_out/p2p.log
python scripts/ab_lib.py ab/libspcg_old.so p3 2 > gpurun_out/ab_p3.log 2>&1; python scripts/ab_lib.py ab/libspcg_old.so p2 2 > gpurun_out/ab_p2.log 2>&1
tail -5 gpurun_out/p2p.log; cat gpurun_out/ab_p3.log gpurun_out/ab_p2.log
