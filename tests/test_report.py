"""CSV layouts match the reference harness (harness.py:124-147)."""

import csv

from paper_1912_03106_b200 import SolverRun, StorageReport
from paper_1912_03106_b200 import report


def _run():
    return SolverRun(converged=True, iterations=2, residual_norms=[1e-3, 1e-8],
                     qoi_changes=[0.5, 1e-9], iteration_seconds=[0.1234, 0.2],
                     setup_seconds=0.5, solve_seconds=0.25,
                     storage=StorageReport(per_level=[4, 6], total=10, estimate=10))


def test_iterations_and_summary(tmp_path):
    report.write_run(tmp_path, _run())
    rows = list(csv.reader(open(tmp_path / "iterations.csv")))
    assert rows[0] == ["iteration", "residual_norm", "qoi_change", "wall_time_s"]
    assert rows[1] == ["1", "0.001", "0.5", "0.123"]
    summ = list(csv.reader(open(tmp_path / "summary.csv")))
    assert summ == [["iterations", "setup_s", "solve_s", "total_s", "converged",
                     "storage_units"], ["2", "0.500", "0.250", "0.750", "true", "10"]]
    assert open(tmp_path / "summary.csv", "rb").read().endswith(b"\n")


def test_scaling_and_compare(tmp_path):
    report.write_scaling_csv(tmp_path / "scaling.csv", 8.0, {1: 4.0, 2: 2.5})
    rows = list(csv.reader(open(tmp_path / "scaling.csv")))
    assert rows == [["p", "total_s", "speedup", "efficiency"],
                    ["1", "4.000", "2.000", "2.000"], ["2", "2.500", "3.200", "1.600"]]
    r = _run()
    report.write_compare_csv(tmp_path / "compare.csv", [("V-gamma1", "none", r),
                                                      ("V-gamma1-sc", "delayed", r)],
                             "V-gamma1")
    rows = list(csv.reader(open(tmp_path / "compare.csv")))
    assert rows[0] == ["variant", "sc_strategy", "iterations", "total_s",
                       "speedup_vs_reference", "converged"]
    assert rows[2][4] == "1.000"
