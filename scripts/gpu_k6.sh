bash scripts/gpu_ab6.sh "$@" 2>&1
SPCG_LIB=ab/lib_allpoll.so SPCG_LIB_LENIENT=1 timeout 300 python scripts/shape_stress.py 10 csr,sympriv,csc 2>&1 | tail -3
