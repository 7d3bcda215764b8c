# engine-6 message protocol check: correctness first, then the A/B timing
timeout 300 python scripts/bimodal.py 20 csr:6,sympriv:6,csc:6 > gpurun_out/mbar_new.log 2>&1; echo bimodal rc=$?
SPCG_LIB=ab/lib_bar.so SPCG_LIB_LENIENT=1 timeout 300 python scripts/bimodal.py 20 csr:6,sympriv:6,csc:6 > gpurun_out/mbar_old.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "pipe or clus or cond or random or reference or engine" > gpurun_out/mbar_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/mbar_tests.log
