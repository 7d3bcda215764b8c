# engine-6 message protocol check: the A/B timing (in-tree vs ab/$1), then correctness
timeout 300 python scripts/bimodal.py 20 csr:6,sympriv:6,csc:6 > gpurun_out/mbar_new.log 2>&1; echo bimodal rc=$?
SPCG_LIB=ab/$1 SPCG_LIB_LENIENT=1 timeout 300 python scripts/bimodal.py 20 csr:6,sympriv:6,csc:6 > gpurun_out/mbar_old.log 2>&1
SPCG_LIB=ab/lib_fine.so SPCG_LIB_LENIENT=1 SPCG_CLUS_DEBUG=gpurun_out/fine.jsonl timeout 300 python scripts/bimodal.py 10 csr:6,sympriv:6 > gpurun_out/fine.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "pipe or clus or cond or random or reference or engine" > gpurun_out/mbar_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/mbar_tests.log
timeout 600 python scripts/clus_stress.py 200 6 > gpurun_out/stress6.log 2>&1; cat gpurun_out/stress6.log
