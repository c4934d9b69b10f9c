"""Generate the parity fixtures in tests/golden/ (run in the survey
container, where /root/reference exists; the GPU box only reads the .npz).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every MGRIT fixture is produced by the REFERENCE's own engine
(pintmg.mgrit.mgrit_solve, /root/reference/pkg/src/pintmg/mgrit.py:797-801)
and sequential stepper (pintmg.problems.sequential_solve, problems.py:319-339)
driving the oracle's 2D problem classes (oracle/fem2d.py) through the
reference's Phi contract.  Phi fixtures are oracle steps on seeded states.
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


def mgrit_case(name, spec, max_iters=50, tol=1e-7, with_solution=True):
    t0 = time.time()
    prob = fem2d.make_problem(spec)
    grid = build_uniform_grid(0.0, spec["tf"], spec["n_steps"])
    mg = spec["mgrit"]
    hier = TimeHierarchy.build(grid, mg["factors"])
    run, sol = mgrit_solve(prob, hier,
                           CycleSpec(kind=mg["kind"], gamma=mg["gamma"],
                                     max_iters=max_iters,
                                     spatial_strategy=mg["spatial_strategy"],
                                     nested_iterations=mg.get("nested_iterations", False)),
                           StoppingCriterion(tolerance=tol))
    seq = sequential_solve(prob, grid.points)
    seq_arr = np.stack([s.field for s in seq.states])
    out = dict(
        spec=json.dumps(spec),
        iterations=run.iterations,
        converged=run.converged,
        history=np.array([run.initial_residual] + list(run.residual_norms)),
        qoi_changes=np.array(run.qoi_changes),
        seq_final=seq_arr[-1],
        seq_norms=np.linalg.norm(seq_arr, axis=1),
        factors=np.array(mg["factors"]),
        max_iters=max_iters,
        tol=tol,
    )
    if with_solution and sol is not None:
        arr = np.stack([s.field for s in sol.states])
        m = mg["factors"][0]
        out["sol_c"] = arr[::m]
        out["sol_norms"] = np.linalg.norm(arr, axis=1)
        out["sol_final"] = arr[-1]
        if getattr(prob, "n_scalars", 0):
            sc = np.stack([s.scalars for s in sol.states])
            out["sol_c_scalars"] = sc[::m]
            out["seq_scalars"] = np.stack([s.scalars for s in seq.states])
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: {run.iterations} iters, converged={run.converged}, "
          f"history={['%.3e' % h for h in out['history']]}  ({time.time() - t0:.1f}s)")


def phi_case(name, spec, B=8, seed=0):
    prob = fem2d.make_problem(spec)
    rng = np.random.default_rng(seed)
    out = {"spec": json.dumps(spec)}
    for g in range(prob.spatial.n_grids):
        n = prob.spatial.size(g)
        U = rng.standard_normal((B, n)) * 1e-3
        t_next = np.sort(rng.uniform(0.0, 0.02, B))
        dt = spec["tf"] / spec["n_steps"] * (1 + np.arange(B) % 3)
        t_prev = t_next - dt
        out[f"u{g}"] = U
        out[f"tp{g}"] = t_prev
        out[f"tn{g}"] = t_next
        out[f"phi{g}"] = prob.step_batch(U, t_prev, t_next, g, False)
        out[f"phis{g}"] = prob.step_batch(U, t_prev, t_next, g, True)
        if g + 1 < prob.spatial.n_grids:
            out[f"R{g}"] = np.stack([prob.spatial.restrict_field(u, g) for u in U])
        if g > 0:
            out[f"P{g}"] = np.stack([prob.spatial.prolong_field(u, g) for u in U])
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: phi fixture with {prob.spatial.n_grids} grids")


def main():
    which = sys.argv[1:] or ["phi", "cfg1", "cfg2s", "cfg2d", "cfg3s", "variants", "surrogate"]
    if "phi" in which:
        phi_case("phi_cfg2_n32", configs.config2(N=32, n_steps=1024, levels=3))
        s = configs.config2(N=32, n_steps=1024, levels=3)
        s["restriction"], s["prolongation"] = "injection", "p1"
        phi_case("phi_cfg2_n32_inj", s)
        phi_case("phi_cfg1", configs.config1())
        phi_case("phi_cfg3_n32", configs.config3(N=32, n_steps=1024, levels=2))
        phi_case("phi_cfg2_n128", configs.config2(N=128, n_steps=2 ** 14, levels=1), B=4)
    if "cfg1" in which:
        mgrit_case("mgrit_cfg1", configs.config1())
    if "cfg2s" in which:
        # config 2 as specified (direct spatial coarsening, 3 grids), reduced
        # mesh / steps: the reference's own algorithm stalls here, so the
        # fixture pins the first iterations of that stall
        mgrit_case("mgrit_cfg2_direct_n32", configs.config2(N=32, n_steps=1024),
                   max_iters=6, with_solution=False)
    if "cfg2d" in which:
        s = configs.config2(N=32, n_steps=1024, levels=3, grids=2, strategy="delayed")
        mgrit_case("mgrit_cfg2_delayed_n32", s)
    if "cfg3s" in which:
        s = configs.config3(N=32, n_steps=256, levels=3, grids=2, strategy="delayed")
        mgrit_case("mgrit_cfg3_delayed_n32", s)


    if "surrogate" in which:
        # f3: rotor angle / speed coupled to the field (problems.py:247-287)
        mgrit_case("mgrit_cfg1_surrogate", configs.with_surrogate(configs.config1()))
        s = configs.config3(N=32, n_steps=256, levels=3, grids=2, strategy="delayed")
        mgrit_case("mgrit_cfg3_surrogate_n32", configs.with_surrogate(s, inertia=2.0,
                                                                      friction=0.3))
    if "variants" in which:
        # F-cycle (mgrit.py:617-626) and nested iterations (mgrit.py:659-675)
        s = configs.config2(N=32, n_steps=1024, levels=3, grids=2, strategy="delayed")
        s["mgrit"]["kind"] = "F"
        mgrit_case("mgrit_cfg2_fcycle_n32", s)
        s = configs.config2(N=32, n_steps=1024, levels=3, grids=2, strategy="delayed")
        s["mgrit"]["nested_iterations"] = True
        mgrit_case("mgrit_cfg2_nested_n32", s)


if __name__ == "__main__":
    main()
