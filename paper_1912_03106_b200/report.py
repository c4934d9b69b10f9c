"""Fixed-schema CSV records of GPU runs, in the reference harness's layouts
(harness.py:1-16, :124-147; pkg/README.md "CSV schemas") so GPU and
reference runs can be compared side by side.  Wall-clock columns carry three
decimals; every other column is written with full precision (repr)."""

import csv
from pathlib import Path

ITERATIONS = ("iteration", "residual_norm", "qoi_change", "wall_time_s")
SUMMARY = ("iterations", "setup_s", "solve_s", "total_s", "converged", "storage_units")
COMPARE = ("variant", "sc_strategy", "iterations", "total_s", "speedup_vs_reference",
           "converged")
SCALING = ("p", "total_s", "speedup", "efficiency")


def _fmt(v):
    return repr(float(v))


def _fmt_time(v):
    return f"{float(v):.3f}"


def _write(path, header, rows):
    with open(path, "w", encoding="utf-8", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(header)
        w.writerows(rows)


def write_iterations_csv(path, run):
    rows = [(k + 1, _fmt(n), _fmt(c), _fmt_time(t)) for k, (n, c, t) in
            enumerate(zip(run.residual_norms, run.qoi_changes, run.iteration_seconds))]
    _write(path, ITERATIONS, rows)


def write_summary_csv(path, run):
    storage = run.storage.total if run.storage is not None else 0
    _write(path, SUMMARY, [(run.iterations, _fmt_time(run.setup_seconds),
                            _fmt_time(run.solve_seconds), _fmt_time(run.total_seconds),
                            "true" if run.converged else "false", storage)])


def write_compare_csv(path, records, reference_label):
    """records: list of (label, sc_strategy, run); speedup vs the run whose
    label is reference_label (total-time ratio)."""
    ref = {lab: run for lab, _, run in records}[reference_label]
    rows = [(lab, sc, run.iterations, _fmt_time(run.total_seconds),
             f"{ref.total_seconds / run.total_seconds:.3f}",
             "true" if run.converged else "false") for lab, sc, run in records]
    _write(path, COMPARE, rows)


def write_scaling_csv(path, sequential_seconds, totals):
    """totals: {p: total seconds}; speedup = sequential / total, efficiency
    = speedup / p (the reference's definitions)."""
    rows = []
    for p in sorted(totals):
        sp = sequential_seconds / totals[p]
        rows.append((p, _fmt_time(totals[p]), f"{sp:.3f}", f"{sp / p:.3f}"))
    _write(path, SCALING, rows)


def write_run(out_dir, run):
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    write_iterations_csv(out / "iterations.csv", run)
    write_summary_csv(out / "summary.csv", run)
