"""Seeded random sweep on the device: arbitrary sparse matrices (empty rows,
rows longer than a tile, n = 1, row-length mixes that take every SpMV body:
thread-per-row, split lines, CSR-stream, CTA-wide long rows) through all four
storages against the oracle; random SPD systems through every CG engine
against the oracle's CG."""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _random_csr(rng, n, kind):
    """kind: 'short' (<= 8/row), 'mid' (9..32/row), 'long' (> 32/row),
    'ragged' (mix incl. empty rows and one row longer than a tile)."""
    from paper_1010_4639_b200.core import build_csr_from_triplets

    if kind == "short":
        lens = rng.integers(1, 9, size=n)
    elif kind == "mid":
        lens = rng.integers(9, 33, size=n)
    elif kind == "long":
        lens = rng.integers(33, 90, size=n)
    else:
        lens = rng.choice([0, 1, 3, 7, 15, 40], size=n)
        if n > 10:
            lens[rng.integers(n)] = min(n, 5000)
    lens = np.minimum(lens, n)
    rows, cols = [], []
    for i, L in enumerate(lens):
        c = rng.choice(n, size=int(L), replace=False)
        rows.append(np.full(int(L), i))
        cols.append(c)
    r = np.concatenate(rows) if rows else np.empty(0, np.int64)
    c = np.concatenate(cols) if cols else np.empty(0, np.int64)
    v = rng.standard_normal(r.size)
    return build_csr_from_triplets((r, c, v), n)


CASES = [(1, "short"), (37, "ragged"), (700, "short"), (700, "mid"), (700, "long"),
         (5000, "ragged"), (20000, "short"), (20000, "mid"), (9000, "long")]


@pytest.mark.parametrize("n,kind", CASES)
def test_random_spmv_all_storages(n, kind):
    from paper_1010_4639_b200 import KernelConfig, spmv_csc, spmv_full, spmv_sym
    from paper_1010_4639_b200.core import build_csr_from_triplets, extract_lower

    rng = np.random.default_rng(n * 7 + len(kind))
    a = _random_csr(rng, n, kind)
    x = rng.standard_normal(n)
    y = spmv_full(a, x)
    yo = O.spmv_full(a.row_start, a.col_idx, a.values, x)
    assert (y == yo).all()                                   # bitwise, sequential rows
    cs = a.to_csc()
    yc = spmv_csc(cs, x)
    scale = max(1.0, float(np.abs(yo).max()))
    assert np.abs(yc - yo).max() <= 1e-12 * scale * max(1, np.diff(a.row_start).max())
    # symmetric half of S = A + A^T (an exactly symmetric operator)
    d = np.arange(n)  # SymHalfMatrix needs a stored diagonal on every row
    r = np.concatenate([a.entry_rows, a.col_idx, d])
    c = np.concatenate([a.col_idx, a.entry_rows, d])
    v = np.concatenate([a.values, a.values, np.ones(n)])
    s_full = build_csr_from_triplets((r, c, v), n)
    s = extract_lower(s_full)
    ys_ref = O.spmv_sym(s.row_start, s.col_idx, s.values, x, accumulation="privatized")
    ysp = spmv_sym(s, x, KernelConfig(accumulation="privatized"))
    assert (ysp == ys_ref).all()                             # bitwise privatized (workers=1)
    ysa = spmv_sym(s, x, KernelConfig(accumulation="atomic"))
    sc = max(1.0, float(np.abs(ys_ref).max()))
    assert np.abs(ysa - ys_ref).max() <= 1e-12 * sc * max(1, np.diff(s_full.row_start).max())


def _storage(a, kind):
    from paper_1010_4639_b200 import KernelConfig, extract_lower

    if kind == "csr":
        return a, KernelConfig()
    if kind == "csc":
        return a.to_csc(), KernelConfig()
    return extract_lower(a), KernelConfig(accumulation="privatized" if kind == "sym_priv"
                                          else "atomic")


def _arrow(n):
    """SPD arrow matrix: dense first row/column (a line longer than a tile),
    tridiagonal body, diagonally dominant."""
    from paper_1010_4639_b200.core import build_csr_from_triplets

    rng = np.random.default_rng(n)
    i = np.arange(1, n)
    w = -rng.uniform(0.1, 1.0, n - 1) / n
    t = -rng.uniform(0.1, 0.5, n - 2)
    rows = np.concatenate([np.zeros(n - 1, int), i, i[:-1], i[1:]])
    cols = np.concatenate([i, np.zeros(n - 1, int), i[1:], i[:-1]])
    vals = np.concatenate([w, w, t, t])
    diag = np.bincount(rows, weights=np.abs(vals), minlength=n) + 0.5
    return build_csr_from_triplets((np.concatenate([rows, np.arange(n)]),
                                    np.concatenate([cols, np.arange(n)]),
                                    np.concatenate([vals, diag])), n)


@pytest.mark.parametrize("engine", [0, 2, 3, 5, 7])
@pytest.mark.parametrize("storage", ["csr", "sym_priv", "sym_atomic", "csc"])
@pytest.mark.parametrize("n,density,seed", [(300, 0.05, 1), (2500, 0.004, 2), (12000, 0.0008, 3),
                                            (6000, -1.0, 4)])
def test_random_spd_all_engines(engine, storage, n, density, seed):
    from paper_1010_4639_b200 import CgOptions, cg_solve
    from paper_1010_4639_b200.genprob import random_spd

    a = random_spd(n, density, seed) if density > 0 else _arrow(n)
    b = np.random.default_rng(seed).standard_normal(n)
    ref = O.cg_solve("csr", a.row_start, a.col_idx, a.values, b)
    m, cfg = _storage(a, storage)
    try:
        r = cg_solve(m, b, opts=CgOptions(record_history=True), cfg=cfg, engine=engine)
    except Exception as e:  # engine 5 may decline unbanded systems, engine 7 the
        # scatter formats; auto never declines
        assert (engine == 5 and "not applicable" in str(e)) or (
            engine == 7 and storage in ("sym_atomic", "csc") and "gather formats" in str(e)), e
        return
    assert abs(r.iterations - ref.iterations) <= max(1, ref.iterations // 100)
    assert np.linalg.norm(r.x - ref.x) / np.linalg.norm(ref.x) <= 1e-8
    assert r.final_relative_residual <= 1e-10


@pytest.mark.parametrize("engine", [0, 2, 3, 5, 7])
def test_degenerate_sizes(engine):
    """n = 0 (empty system: b = 0 -> x = [] converged, as solver.py:109-118)
    and n = 1 through every engine and storage."""
    from paper_1010_4639_b200 import CgOptions, cg_solve, spmv_full
    from paper_1010_4639_b200.core import build_csr_from_triplets

    e = np.empty(0, dtype=np.int64)
    a0 = build_csr_from_triplets((e, e, np.empty(0)), 0)
    r0 = cg_solve(a0, np.empty(0), engine=engine)
    assert r0.iterations == 0 and r0.converged and r0.x.shape == (0,)
    assert spmv_full(a0, np.empty(0)).shape == (0,)
    a1 = build_csr_from_triplets((np.array([0]), np.array([0]), np.array([4.0])), 1)
    for kind in ("csr", "sym_priv") if engine == 7 else ("csr", "sym_priv", "sym_atomic", "csc"):
        m, cfg = _storage(a1, kind)
        r1 = cg_solve(m, np.array([2.0]), opts=CgOptions(record_history=True), cfg=cfg,
                      engine=engine)
        assert r1.iterations == 1 and r1.converged and r1.x[0] == 0.5, (kind, r1)


@pytest.mark.parametrize("storage", ["csr", "sym_priv"])
def test_row_sums_modes_long_rows(storage):
    """27-point rows (split-line tiles) in the per-pass engine: the default
    reassociated long-row sums and KernelConfig(row_sums="sequential") both
    follow the reference CG; each is deterministic run to run."""
    from paper_1010_4639_b200 import CgOptions, KernelConfig, cg_solve, extract_lower
    from paper_1010_4639_b200.genprob import rhs_for, stencil27

    a = stencil27(20, 18, 16)
    b, _ = rhs_for(a, seed=4)
    ref = O.cg_solve("csr", a.row_start, a.col_idx, a.values, b)
    m = a if storage == "csr" else extract_lower(a)
    for mode in ("auto", "sequential"):
        cfg = KernelConfig(accumulation="privatized", row_sums=mode)
        r1 = cg_solve(m, b, opts=CgOptions(record_history=True), cfg=cfg, engine=2)
        r2 = cg_solve(m, b, opts=CgOptions(record_history=True), cfg=cfg, engine=2)
        assert r1.iterations == r2.iterations and (r1.x == r2.x).all()
        assert abs(r1.iterations - ref.iterations) <= max(1, ref.iterations // 100)
        assert np.linalg.norm(r1.x - ref.x) / np.linalg.norm(ref.x) <= 1e-8
    with pytest.raises(ValueError):
        KernelConfig(row_sums="fast")


@pytest.mark.parametrize("engine", [0, 2, 7])
@pytest.mark.parametrize("storage", ["csr", "sym_priv", "sym_atomic", "csc"])
def test_streaming_engines_all_storages(engine, storage):
    """A system too large for the resident kernels (auto routes it to the
    per-pass streaming engine) in every storage, against the reference CG;
    engines 1 and 4 of round 1 are gone and rejected."""
    from paper_1010_4639_b200 import CgOptions, cg_solve
    from paper_1010_4639_b200.genprob import poisson3d, rhs_for

    a = poisson3d(48, 48, 64)
    b, _ = rhs_for(a, seed=6)
    ref = O.cg_solve("csr", a.row_start, a.col_idx, a.values, b)
    m, cfg = _storage(a, storage)
    assert m.device().info()["ntiles"] > 2 * 148
    if engine == 7 and storage in ("sym_atomic", "csc"):
        with pytest.raises(Exception, match="gather formats"):
            cg_solve(m, b, cfg=cfg, engine=engine)
        return
    r = cg_solve(m, b, opts=CgOptions(record_history=True), cfg=cfg, engine=engine)
    assert abs(r.iterations - ref.iterations) <= max(1, ref.iterations // 100)
    assert np.linalg.norm(r.x - ref.x) / np.linalg.norm(ref.x) <= 1e-8
    assert r.final_relative_residual <= 1e-10


@pytest.mark.parametrize("engine", [1, 4, 8, -1])
def test_removed_engines_are_rejected(engine):
    from paper_1010_4639_b200 import cg_solve
    from paper_1010_4639_b200.genprob import poisson2d

    a = poisson2d(8, 8)
    with pytest.raises(ValueError, match="engine must be"):
        cg_solve(a, np.ones(a.n), engine=engine)


@pytest.mark.parametrize("dims,engine_expected", [((512, 512), 7), ((1448, 1448), 2)])
def test_auto_routes_midsize_csr(dims, engine_expected):
    """Auto on full CSR that does not fit on chip: engine 7 (one persistent
    streamed launch) up to ~1 M rows, the per-pass engine beyond; both follow
    the serial reference CG's iteration count (capped) and each other's x."""
    from paper_1010_4639_b200 import CgOptions, cg_solve
    from paper_1010_4639_b200.genprob import poisson2d

    a = poisson2d(*dims)
    b = np.random.default_rng(11).standard_normal(a.n)
    r0 = cg_solve(a, b, opts=CgOptions(max_iter=300, record_history=True))
    assert r0.engine_info["engine"] == engine_expected
    other = 2 if engine_expected == 7 else 7
    r1 = cg_solve(a, b, opts=CgOptions(max_iter=300, record_history=True), engine=other)
    assert r0.iterations == r1.iterations == 300
    assert np.linalg.norm(r0.x - r1.x) / np.linalg.norm(r1.x) <= 1e-12
    assert np.allclose(r0.residual_history, r1.residual_history, rtol=1e-6)
