"""A/B two builds of the library on the same box, interleaved:
    python scripts/ab_lib.py ab/libspcg_old.so [workload] [rounds]
Each round runs bench.py (no secondary / cpu baseline) once per library via
SPCG_LIB and prints the dominant-kernel time, the step time and the clock."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
libs = {"B": str(ROOT / "paper_1010_4639_b200/_lib/libspcg_b200.so"), "A": sys.argv[1]}
wl = sys.argv[2] if len(sys.argv) > 2 else "p3"
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 2
for r in range(rounds):
    for name in ("A", "B"):
        env = dict(os.environ, SPCG_LIB=libs[name], SPCG_LIB_LENIENT="1")
        p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--no-secondary",
                            "--no-cpu-baseline", "--workload", wl, "--steps", "3", "--warmup", "2"],
                           env=env, capture_output=True, text=True)
        try:
            d = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][-1])
            print(json.dumps({"lib": name, "round": r, "kernel_ms": d["roofline"]["kernel_ms"],
                              "frac": d["roofline"]["frac"], "ms_per_step": d["ms_per_step"],
                              "us_it": d["roofline_iteration"]["us_per_iteration"],
                              "sm_mhz": d["clocks"]["sm_mhz"]}), flush=True)
        except Exception:  # noqa: BLE001
            print(name, "failed", p.stderr[-800:], flush=True)
