"""Full-size parity fixtures (run where /root/reference exists; the GPU box
only reads the .npz).

    PYTHONPATH=/root/reference/pkg/src OMP_NUM_THREADS=1 \
        python tests/golden/make_golden_full.py cfg2_full

Like make_golden.py, every MGRIT run here is the REFERENCE's own engine
(pintmg.mgrit.mgrit_solve, /root/reference/pkg/src/pintmg/mgrit.py:797-801)
and sequential stepper (pintmg.problems.sequential_solve,
problems.py:319-339) driving the oracle's 2D problem classes.  The states
at these sizes are too large to commit whole (config 2: 1,025 C-points x
16,129 DOFs = 132 MB), so a fixture keeps

  * the residual history and iteration count (the north-star's 1e-8 gate),
  * the L2 norm of every C-point state of the MGRIT iterate and of the
    sequential solution,
  * a handful of whole C-point states (sampled evenly, first and last
    included) of both, and the final sequential state.

Cases:
  cfg2_full    config 2 at its stated size (127^2 unknowns, 2^14 steps,
               3 levels, m = 16), delayed spatial coarsening --
               the bench's config-2 leg.
  cfg4shape    the 4-level [16, 16, 16] cycle of config 4 on config 2's
               127^2 mesh and 2^14 steps, delayed coarsening.
  cfg3_n64     config 3 (Brauer nonlinearity, damped Newton) on a 63^2 mesh
               with 2^12 steps, 3 levels, delayed coarsening.
  cfg2_direct_n128  config 2 literal (direct coarsening, 3 grids), the first
               6 iterations at full size: the stall DESIGN.md 2 documents.
"""

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from pintmg.mgrit import CycleSpec, StoppingCriterion, mgrit_solve  # noqa: E402
from pintmg.problems import sequential_solve  # noqa: E402
from pintmg.time_hierarchy import TimeHierarchy, build_uniform_grid  # noqa: E402

from oracle import fem2d  # noqa: E402
from paper_1912_03106_b200 import configs  # noqa: E402

N_SAMPLES = 8


def sample_idx(k_points):
    return np.unique(np.linspace(0, k_points - 1, N_SAMPLES).round().astype(np.int64))


def full_case(name, spec, max_iters=50, tol=1e-7, with_solution=True, with_seq=True):
    t0 = time.time()
    prob = fem2d.make_problem(spec)
    grid = build_uniform_grid(0.0, spec["tf"], spec["n_steps"])
    mg = spec["mgrit"]
    m = mg["factors"][0]
    hier = TimeHierarchy.build(grid, mg["factors"])
    run, sol = mgrit_solve(prob, hier,
                           CycleSpec(kind=mg["kind"], gamma=mg["gamma"],
                                     max_iters=max_iters,
                                     spatial_strategy=mg["spatial_strategy"],
                                     nested_iterations=mg.get("nested_iterations", False)),
                           StoppingCriterion(tolerance=tol))
    t_mg = time.time() - t0
    out = dict(
        spec=json.dumps(spec),
        iterations=run.iterations,
        converged=run.converged,
        history=np.array([run.initial_residual] + list(run.residual_norms)),
        factors=np.array(mg["factors"]),
        max_iters=max_iters,
        tol=tol,
        mgrit_seconds=t_mg,
    )
    if with_solution and sol is not None:
        c_states = [s.field for s in sol.states[::m]]
        idx = sample_idx(len(c_states))
        out["sol_c_norms"] = np.array([np.linalg.norm(u) for u in c_states])
        out["sol_c_idx"] = idx
        out["sol_c_samples"] = np.stack([c_states[i] for i in idx])
        del c_states
    del sol
    if with_seq:
        t1 = time.time()
        seq = sequential_solve(prob, grid.points)
        c_seq = [s.field for s in seq.states[::m]]
        idx = sample_idx(len(c_seq))
        out["seq_c_norms"] = np.array([np.linalg.norm(u) for u in c_seq])
        out["seq_c_idx"] = idx
        out["seq_c_samples"] = np.stack([c_seq[i] for i in idx])
        out["seq_final"] = seq.states[-1].field
        out["seq_seconds"] = time.time() - t1
        del seq, c_seq
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: {run.iterations} iters, converged={run.converged}, "
          f"history={['%.3e' % h for h in out['history']]}  "
          f"(mgrit {t_mg:.0f}s, total {time.time() - t0:.0f}s)", flush=True)


CASES = {
    "cfg2_full": lambda: full_case(
        "mgrit_cfg2_full", configs.config2(grids=2, strategy="delayed")),
    "cfg4shape": lambda: full_case(
        "mgrit_cfg4shape_n128",
        configs.config2(N=128, n_steps=2 ** 14, levels=4, grids=2, strategy="delayed")),
    "cfg3_n64": lambda: full_case(
        "mgrit_cfg3_n64",
        configs.config3(N=64, n_steps=2 ** 12, levels=3, grids=2, strategy="delayed")),
    "cfg2_direct_n128": lambda: full_case(
        "mgrit_cfg2_direct_n128", configs.config2(), max_iters=6,
        with_solution=False, with_seq=False),
}


def main():
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()


if __name__ == "__main__":
    main()
