for m in 1 0 1 0; do echo "== sort $m"; SPCG_CLUS_SORT=$m timeout 300 python scripts/sort_ab.py 2>&1 | tail -1; done
