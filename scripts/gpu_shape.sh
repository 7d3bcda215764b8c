# engine-6 grid shape A/B (dev env knobs of host_cluster.cuh)
C="csr:6,sympriv:6"
echo "== default"; timeout 300 python scripts/bimodal.py 20 $C 2>&1 | cut -c1-110
echo "== csz16"; SPCG_CLUS_CSZ=16 timeout 300 python scripts/bimodal.py 20 $C 2>&1 | cut -c1-110
echo "== csz4"; SPCG_CLUS_CSZ=4 timeout 300 python scripts/bimodal.py 20 $C 2>&1 | cut -c1-110
for k in 6 10 12 18; do echo "== K$k"; SPCG_CLUS_K=$k timeout 300 python scripts/bimodal.py 20 $C 2>&1 | cut -c1-110; done
echo "== csz16 K6"; SPCG_CLUS_CSZ=16 SPCG_CLUS_K=6 timeout 300 python scripts/bimodal.py 20 $C 2>&1 | cut -c1-110
echo "== csz16 K9"; SPCG_CLUS_CSZ=16 SPCG_CLUS_K=9 timeout 300 python scripts/bimodal.py 20 $C 2>&1 | cut -c1-110
SPCG_TRACE=1 SPCG_CLUS_CSZ=16 timeout 300 python scripts/bimodal.py 1 csr:6 2>&1 | grep "spcg trace" | head -2
