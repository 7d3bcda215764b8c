# A/B of engine-6 builds on one box: in-tree vs each ab/<lib> given, interleaved twice
for r in 1 2; do
  echo "== in-tree"; timeout 300 python scripts/bimodal.py 20 ${CASES:-csr:6,sympriv:6,csc:6} 2>&1 | cut -c1-120
  for l in "$@"; do
    echo "== $l"; SPCG_LIB=ab/$l SPCG_LIB_LENIENT=1 timeout 300 python scripts/bimodal.py 20 ${CASES:-csr:6,sympriv:6,csc:6} 2>&1 | cut -c1-120
  done
done
