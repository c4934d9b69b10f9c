"""Time-to-solution of BASELINE configs 1-3 at full size on one GPU (dev tool).

usage: python tools/probe_configs.py cfg1|cfg2|cfg2-direct|cfg3|cfg3-window|cfg4[-window][-delayed] [max_iters]
"""
import json, sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1912_03106_b200 import (GpuFemProblem, CycleSpec, StoppingCriterion, TimeHierarchy,
                                   build_uniform_grid, MgritSolver, sequential_solve, configs, build)
build.build()
name = sys.argv[1]
max_iters = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 50
if name == "cfg1":
    spec = configs.config1()
elif name == "cfg2":
    spec = configs.config2(grids=2, strategy="delayed")
elif name == "cfg2-direct":
    spec = configs.config2()
elif name == "cfg3":
    spec = configs.config3(grids=2, strategy="delayed")
elif name == "cfg3-window":
    spec = configs.config3(n_steps=2 ** 10, grids=2, strategy="delayed")
elif name.startswith("cfg4"):
    # cfg4, cfg4-window (2^12 steps), cfg4-delayed, cfg4-window-delayed
    win = "window" in name
    kw = dict(grids=2, strategy="delayed") if "delayed" in name else {}
    spec = configs.config4(n_steps=2 ** 12 if win else 2 ** 16, **kw)
    if win:
        spec["tf"] = spec["tf"] * 2 ** 12 / 2 ** 16
else:
    raise SystemExit(name)
if "merge" in sys.argv[2:]:
    spec["inner"]["dt_merge_rtol"] = 1e-12
prob = GpuFemProblem(spec)
mg = spec["mgrit"]
grid = build_uniform_grid(0.0, spec["tf"] * spec["n_steps"] / 2 ** 14 if name == "cfg3-window" else spec["tf"], spec["n_steps"])
solver = MgritSolver(prob, TimeHierarchy.build(grid, mg["factors"]),
                     CycleSpec(kind="V", gamma=1, max_iters=max_iters,
                               spatial_strategy=mg["spatial_strategy"]),
                     StoppingCriterion(tolerance=mg["tolerance"]))
t0 = time.perf_counter()
run, _ = solver.solve(gather_solution=False)
torch.cuda.synchronize()
t = time.perf_counter() - t0
st = prob.total_stats()
print(json.dumps({"config": name, "n": prob.spatial.size(0), "n_steps": spec["n_steps"],
                  "inner": prob.inner, "nonlinear": prob.nonlinear,
                  "wall_s": t, "solve_s": run.solve_seconds, "iterations": run.iterations,
                  "converged": run.converged, "failure": run.failure,
                  "history": [run.initial_residual] + run.residual_norms,
                  "phi_columns": run.phi_columns, "inner_iters": st["column_iters"],
                  "newton_iters": st["newton_iters"],
                  "step_dof_per_s": spec["n_steps"] * prob.spatial.size(0) / t,
                  "dt_merge_rtol": spec["inner"].get("dt_merge_rtol", 0.0),
                  "gpu_mem_used_gb": (lambda f: (f[1] - f[0]) / 1e9)(torch.cuda.mem_get_info())}),
      flush=True)
