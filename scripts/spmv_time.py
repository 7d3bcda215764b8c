"""Dev helper: standalone SpMV timing on the generated stencil matrices.
python scripts/spmv_time.py [Q27 Q27P Q27F P3 P2]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1010_4639_b200.device import DeviceMatrix  # noqa: E402
from scripts.probe import spmv_time  # noqa: E402

CFG = {"Q27": ("stencil27", (256, 256, 256), "scsr", 0), "Q27P": ("stencil27", (256, 256, 256), "scsr", 1),
       "Q27F": ("stencil27", (256, 256, 256), "csr", 1), "P3": ("poisson3d", (400, 400, 400), "csr", 1),
       "P2": ("poisson2d", (4096, 4096), "csr", 1)}
for c in sys.argv[1:] or ["Q27"]:
    kind, dims, fmt, acc = CFG[c]
    dm = DeviceMatrix.generate(kind, dims, fmt)
    print(json.dumps({"cfg": c, "spmv_ms": [round(spmv_time(dm, acc, dm.n), 4) for _ in range(3)]}), flush=True)
    dm.close()
