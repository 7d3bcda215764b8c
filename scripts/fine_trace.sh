# engine-6 sub-phase timers (A/B build ab/lib_fine.so, -DSPCG_PIPE_FINE=1)
python scripts/bimodal.py 20 csr:6,sympriv:6 > gpurun_out/fine_base.log 2>&1
SPCG_LIB=ab/lib_fine.so SPCG_LIB_LENIENT=1 SPCG_CLUS_DEBUG=gpurun_out/fine.jsonl python scripts/bimodal.py 20 csr:6,sympriv:6 > gpurun_out/fine.log 2>&1
