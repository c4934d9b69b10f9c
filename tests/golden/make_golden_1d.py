"""Fixtures from the reference's OWN 1D problem and engine (run where
/root/reference exists; tests only read the .npz):

    python tests/golden/make_golden_1d.py

* ref1d_step: `LinearDiffusionProblem.step` (problems.py:138-146) on seeded
  states -- the setting of the reference's test_problems.py:56-66 -- plus a
  mixed-dt batch.
* ref1d_mgrit: the reference engine (`pintmg.mgrit.mgrit_solve`) and
  `sequential_solve` on `LinearDiffusionProblem(31)` with the default
  PwmSource, 64 steps, two-level m = 4, gamma 0 and 1, tolerance 1e-12 -- the
  setting of test_acceptance.py:47-62 -- and a 5-level [2, 2, 2, 2] V-cycle on
  256 steps (the hierarchy shape of test_acceptance.py:248-267).
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from pintmg.excitation import PwmSource  # noqa: E402
from pintmg.mgrit import CycleSpec, StoppingCriterion, mgrit_solve  # noqa: E402
from pintmg.problems import LinearDiffusionProblem, sequential_solve  # noqa: E402
from pintmg.state import BlockState  # noqa: E402
from pintmg.time_hierarchy import TimeHierarchy, build_uniform_grid  # noqa: E402


def step_fixture():
    n, nu, sigma = 31, 0.7, 1.3
    prob = LinearDiffusionProblem(n, diffusivity=nu, mass_coeff=sigma, excitation=PwmSource())
    rng = np.random.default_rng(0)
    B = 12
    U = rng.normal(size=(B, n))
    t_prev = 0.001 + 0.0007 * np.arange(B)
    dts = np.array([1e-3, 1e-3, 5e-4, 1e-3, 2.5e-4, 5e-4, 1e-3, 1e-4, 1e-3, 5e-4, 1e-3, 2e-3])
    t_next = t_prev + dts
    out = np.stack([prob.step(BlockState(U[b]), float(t_prev[b]), float(t_next[b]))[0].field
                    for b in range(B)])
    out_smooth = np.stack([prob.step(BlockState(U[b]), float(t_prev[b]), float(t_next[b]),
                                     smooth=True)[0].field for b in range(B)])
    src = np.array([prob.excitation.value(float(t)) for t in t_next])
    src_s = np.array([prob.excitation.smooth_value(float(t)) for t in t_next])
    np.savez_compressed(os.path.join(HERE, "ref1d_step.npz"), n=n, diffusivity=nu,
                        mass_coeff=sigma, U=U, t_prev=t_prev, t_next=t_next, out=out,
                        out_smooth=out_smooth, src=src, src_smooth=src_s,
                        shape=prob._shapes[0], weights=prob.loss_weights(0))


def mgrit_fixture():
    prob = LinearDiffusionProblem(31, diffusivity=1.0, excitation=PwmSource(), source="sine")
    grid = build_uniform_grid(0.0, 0.02, 64)
    seq = sequential_solve(prob, grid.points)
    seq_arr = np.stack([s.field for s in seq.states])
    hier = TimeHierarchy.build(grid, [4])
    out = dict(times=grid.points, seq=seq_arr)
    for gamma, cap in ((0, 16), (1, 8)):
        run, sol = mgrit_solve(prob, hier, CycleSpec(kind="two-level", gamma=gamma, max_iters=cap),
                               StoppingCriterion(tolerance=1e-12))
        out[f"hist_g{gamma}"] = np.array([run.initial_residual] + list(run.residual_norms))
        out[f"iters_g{gamma}"] = run.iterations
        out[f"sol_g{gamma}"] = np.stack([s.field for s in sol.states])
    grid5 = build_uniform_grid(0.0, 0.02, 256)
    hier5 = TimeHierarchy.build(grid5, [2, 2, 2, 2])
    run, sol = mgrit_solve(prob, hier5, CycleSpec(kind="V", gamma=1, max_iters=30),
                           StoppingCriterion(tolerance=1e-10))
    out["times5"] = grid5.points
    out["hist5"] = np.array([run.initial_residual] + list(run.residual_norms))
    out["iters5"] = run.iterations
    out["sol5"] = np.stack([s.field for s in sol.states])
    np.savez_compressed(os.path.join(HERE, "ref1d_mgrit.npz"), **out)
    print("two-level iterations", out["iters_g0"], out["iters_g1"], "five-level", out["iters5"])


if __name__ == "__main__":
    step_fixture()
    mgrit_fixture()
