# engine-6 register-row variant A/B (SPCG_PIPE_REG=0 turns it off) + correctness
for r in 1 2; do
  echo "== reg"; timeout 300 python scripts/bimodal.py 20 csr:6,sympriv:6,csc:6 2>&1 | cut -c1-110
  echo "== noreg"; SPCG_PIPE_REG=0 timeout 300 python scripts/bimodal.py 20 csr:6,sympriv:6,csc:6 2>&1 | cut -c1-110
done
for k in 6 8; do echo "== K$k"; SPCG_CLUS_K=$k timeout 300 python scripts/shape_stress.py 10 csr,sympriv,csc 2>&1 | tail -3; done
timeout 900 python -m pytest tests -m gpu -x -q -k "pipe or clus or cond or random or reference" 2>&1 | tail -2
timeout 600 python scripts/clus_stress.py 100 6 2>&1 | grep engine
