for r in 1 2; do
for c in P2 P3 Q27 Q27P; do
  echo "== in-tree $c"; timeout 300 python scripts/phase_split.py $c 100 2>&1 | tail -1
  echo "== head $c"; SPCG_LIB=ab/lib_head.so SPCG_LIB_LENIENT=1 timeout 300 python scripts/phase_split.py $c 100 2>&1 | tail -1
done
done
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
