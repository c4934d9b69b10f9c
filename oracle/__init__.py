"""CPU oracle for the batched-Phi MGRIT hot path -- TEST INFRASTRUCTURE ONLY.

Nothing in the product package (`paper_1912_03106_b200`) imports this
package.  Only `tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` /
`--impl reference` legs of `bench.py` may use it, and only as the checker or
as the timed CPU baseline -- never as the thing measured for the GPU arm.

What it restates (own code, following the reference's algorithm):

* `excitation.py`  -- /root/reference/pkg/src/pintmg/excitation.py:26-92
* `state.py`       -- /root/reference/pkg/src/pintmg/state.py:17-164
* `time_hierarchy.py` -- /root/reference/pkg/src/pintmg/time_hierarchy.py:50-175
* `spatial2d.py`   -- 2D tensor-product analogue of spatial.py:20-106
* `fem2d.py`       -- the 2D P1 magnetoquasistatic Phi that BASELINE.json's
  configs name.  The reference has no 2D operator, so the
  problem classes follow the reference's 1D ones line by line in structure:
  linear step = problems.py:122-146 (banded Cholesky via scipy's
  cholesky_banded / cho_solve_banded, cached per (grid, float(dt))), damped
  Newton = problems.py:201-244, sequential oracle = problems.py:319-339.
* `mgrit.py`       -- the MGRIT-FAS engine, mgrit.py:290-801, restated for a
  single worker with every sweep batched over the C-intervals (the same order
  of operations; every sweep starts from pre-sweep C-values).

Pinning: tests/golden/ holds fixtures produced by the *reference's own*
`MgritSolver`/`sequential_solve` (imported from /root/reference in the
survey container by tests/golden/make_golden.py) driving these problem
classes; tests/test_oracle.py checks this package against them and against
the reference tests' closed-form vectors.
"""
