# engine-6 A/B (in-tree vs ab/<lib>) + correctness
bash scripts/gpu_ab6.sh "$@" 2>&1
for k in 6 8; do echo "== K$k"; SPCG_CLUS_K=$k timeout 300 python scripts/shape_stress.py 10 csr,sympriv,csc 2>&1 | tail -3; done
timeout 900 python -m pytest tests -m gpu -x -q -k "pipe or clus or cond or random or reference" 2>&1 | tail -2
timeout 600 python scripts/clus_stress.py 100 6 2>&1 | grep engine
