"""Conditioning sweep table (engines x systems) vs the reference CG (oracle).

    python scripts/cond_sweep.py > gpurun_out/cond_sweep.jsonl

For every system: the reference CG restated in C at workers = host cores
(x_ref) and two other reassociations of the SAME reference algorithm
(workers = 1, and the symmetric-half storage with the atomic scatter) give
the spread that fp64 reassociation alone produces; then every engine's
iterations, ||x - x_ref|| / ||x_ref|| and true final residual."""

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_1010_4639_b200 import CgOptions, KernelConfig, cg_solve, extract_lower  # noqa: E402
from paper_1010_4639_b200.genprob import fem_mesh, poisson2d, random_spd, rhs_for  # noqa: E402


def systems():
    for s in (1.0, 0.1, 0.01, 1e-3, 1e-4, 1e-5):
        yield f"fem_shift{s:g}", fem_mesh(shift=s), 1e-10
    for side in (256, 448):
        yield f"poisson2d_{side}", poisson2d(side, side), 1e-10
    yield "poisson2d_320_tol1e-12", poisson2d(320, 320), 1e-12
    yield "fem_rand", random_spd(30880, 418918 / 30880 ** 2, seed=1), 1e-10


def main():
    eng = [int(e) for e in sys.argv[1:]] or [0, 2, 3, 5, 6]
    for name, a, tol in systems():
        b, _ = rhs_for(a, seed=1)
        cores = O.host_cores()
        ref = O.cg_solve("csr", a.row_start, a.col_idx, a.values, b, tol=tol, workers=cores)
        nx = np.linalg.norm(ref.x)
        r1 = O.cg_solve("csr", a.row_start, a.col_idx, a.values, b, tol=tol, workers=1)
        s = extract_lower(a)
        ra = O.cg_solve("sym", s.row_start, s.col_idx, s.values, b, tol=tol, workers=cores,
                        accumulation="atomic")
        spread = max(np.linalg.norm(r1.x - ref.x), np.linalg.norm(ra.x - ref.x)) / nx
        row = {"system": name, "n": a.n, "ref_it": ref.iterations, "ref_true": ref.final_relative_residual,
               "ref_spread": spread, "ref_its_variants": [r1.iterations, ra.iterations], "engines": {}}
        for e in eng:
            for st in ("csr", "sym_priv"):
                m = a if st == "csr" else s
                cfg = KernelConfig(accumulation="privatized")
                try:
                    t0 = time.perf_counter()
                    r = cg_solve(m, b, opts=CgOptions(tol=tol), cfg=cfg, engine=e)
                    row["engines"][f"{e}/{st}"] = {
                        "it": r.iterations, "conv": r.converged,
                        "err": float(np.linalg.norm(r.x - ref.x) / nx),
                        "true": r.final_relative_residual, "s": round(time.perf_counter() - t0, 4)}
                except Exception as ex:  # noqa: BLE001
                    row["engines"][f"{e}/{st}"] = {"error": str(ex)[:120]}
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
