#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_clus.py tests/test_gpu_pipe.py tests/test_gpu_cg1.py tests/test_gpu_conditioning.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/check.log 2>&1; echo pytest_exit=$? >> gpurun_out/check.log
N=${N:-100} CASES=${CASES:-csr:0,csc:0,sympriv:0,symatom:0,csr:6,csr:3,csr:5} LIBS="paper_1010_4639_b200/_lib/libspcg_b200.so" bash scripts/ab_bimodal.sh > gpurun_out/ab_bimodal7.log 2>&1
tail -3 gpurun_out/check.log; cat gpurun_out/ab_bimodal7.log
