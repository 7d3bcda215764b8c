"""The Table-I harness in the reference's report schema (spcg bench.py,
tests/test_cli_bench.py::TestBench) on the device."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _system(seed=2, dims=(6, 6)):
    from paper_1010_4639_b200.genprob import poisson2d
    from paper_1010_4639_b200.matio import LinearSystem

    a = poisson2d(*dims)
    x = np.random.default_rng(seed).standard_normal(a.n)
    return LinearSystem(matrix=a, b=a.to_dense() @ x, x_ref=x)


def test_text_rows_present():
    from paper_1010_4639_b200.table1 import run_bench

    out = run_bench(_system(), workers_list=[1, 2], reps=3).to_text()
    for row in ("dotProd", "AXPY", "SpMV", "SpMV(sym)", "CG/ # int"):
        assert row in out
    assert "CG/ # int (full)" in out and "CG/ # int (sym)" in out and "CG/ # int (csc)" in out
    assert "backend=cuda" in out


def test_workers_one_speedups_are_unity():
    from paper_1010_4639_b200.table1 import run_bench

    report = run_bench(_system(), workers_list=[1], reps=3)
    assert all(r.speedup == 1.0 for r in report.ops)
    assert all(r.speedup == 1.0 for r in report.cg)
    assert all(c.converged for c in report.cg)


def test_reps_below_three_rejected():
    from paper_1010_4639_b200.table1 import run_bench

    with pytest.raises(ValueError):
        run_bench(_system(), reps=2)


@pytest.mark.parametrize("device_vectors", [True, False])
def test_harness_does_not_mutate_input_and_round_trips(device_vectors):
    from paper_1010_4639_b200.table1 import BenchReport, run_bench, system_checksum

    system = _system()
    before = system_checksum(system)
    report = run_bench(system, workers_list=[1, 2], reps=3, device_vectors=device_vectors)
    assert system_checksum(system) == before
    assert BenchReport.from_json(report.to_json()) == report
    back = BenchReport.from_csv(report.to_csv())
    assert back.ops == report.ops and back.cg == report.cg


def test_deterministic_report_fields():
    from paper_1010_4639_b200.table1 import run_bench

    r1 = run_bench(_system(), workers_list=[1], reps=3, accumulation="privatized")
    r2 = run_bench(_system(), workers_list=[1], reps=3, accumulation="privatized")
    assert [(c.iterations, c.final_relative_residual) for c in r1.cg] == [
        (c.iterations, c.final_relative_residual) for c in r2.cg]


def test_sym_input_also_benches():
    from paper_1010_4639_b200.core import extract_lower
    from paper_1010_4639_b200.matio import LinearSystem
    from paper_1010_4639_b200.table1 import run_bench

    s = _system()
    out = run_bench(LinearSystem(matrix=extract_lower(s.matrix), b=s.b), reps=3).to_text()
    assert "input=sym" in out
