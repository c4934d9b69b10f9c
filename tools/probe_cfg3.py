"""Config 3 (nonlinear, 127^2, 2^14 steps, 3 levels, delayed coarsening) on one
GPU: time-to-solution, Newton / CG counts, band-kernel profile (dev tool).
usage: python tools/probe_cfg3.py [n_steps] [profile]"""
import json, sys, time
import torch
sys.path.insert(0, '.')
from paper_1912_03106_b200 import (GpuFemProblem, CycleSpec, StoppingCriterion, TimeHierarchy,
                                   build_uniform_grid, MgritSolver, configs, build)
build.build()
n_steps = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 2 ** 14
spec = configs.config3(n_steps=n_steps, grids=2, strategy="delayed")
tf = spec["tf"] * n_steps / 2 ** 14
prob = GpuFemProblem(spec)
mg = spec["mgrit"]
grid = build_uniform_grid(0.0, tf, n_steps)


def make():
    return MgritSolver(prob, TimeHierarchy.build(grid, mg["factors"]),
                       CycleSpec(kind="V", gamma=1, max_iters=50,
                                 spatial_strategy=mg["spatial_strategy"]),
                       StoppingCriterion(tolerance=mg["tolerance"]))


s = make()
t0 = time.perf_counter()
run, _ = s.solve(gather_solution=False)
torch.cuda.synchronize()
cold = time.perf_counter() - t0
prob.total_stats(reset=True)
t0 = time.perf_counter()
run, _ = s.solve(gather_solution=False)
torch.cuda.synchronize()
warm = time.perf_counter() - t0
st = prob.total_stats()
out = {"n_steps": n_steps, "cold_s": cold, "warm_s": warm, "iterations": run.iterations,
       "history": [run.initial_residual] + run.residual_norms, "failure": run.failure,
       "phi_calls": run.phi_calls, "phi_columns": run.phi_columns,
       "batched_cg_iters": st["column_iters"], "newton_iters": st["newton_iters"],
       "launches": st["launches"],
       "step_dof_per_s": n_steps * prob.spatial.size(0) / warm}
if "profile" in sys.argv:
    prob.profile(True)
    t0 = time.perf_counter()
    s.solve(gather_solution=False)
    torch.cuda.synchronize()
    out["profiled_s"] = time.perf_counter() - t0
    out["kernels"] = {k["name"]: [k["launches"], round(k["total_ms"], 1)]
                      for k in prob.profile_read(reset=True) if k["launches"]}
    prob.profile(False)
print(json.dumps(out))
