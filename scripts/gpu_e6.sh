# engine-6 A/B (in-tree vs ab/<lib>) + correctness of the ab lib
bash scripts/gpu_ab6.sh "$@" 2>&1
L=ab/$1
for k in 6 8; do echo "== K$k"; SPCG_LIB=$L SPCG_LIB_LENIENT=1 SPCG_CLUS_K=$k timeout 300 python scripts/shape_stress.py 10 csr,sympriv,csc 2>&1 | tail -3; done
SPCG_LIB=$L SPCG_LIB_LENIENT=1 timeout 900 python -m pytest tests -m gpu -x -q -k "pipe or cond or reference" 2>&1 | tail -2
SPCG_LIB=$L SPCG_LIB_LENIENT=1 timeout 600 python scripts/clus_stress.py 100 6 2>&1 | grep engine
