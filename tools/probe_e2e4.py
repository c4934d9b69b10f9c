"""Config 4 end to end (fresh problem + solver + first solve), parts (dev)."""
import sys, time
import torch
sys.path.insert(0, '.')
from paper_1912_03106_b200 import (GpuFemProblem, CycleSpec, StoppingCriterion, TimeHierarchy,
                                   build_uniform_grid, MgritSolver, configs, build)
build.build()
spec = configs.config4(grids=2, strategy="delayed")
mg = spec["mgrit"]
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter()
    prob = GpuFemProblem(spec)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    grid = build_uniform_grid(0.0, spec["tf"], spec["n_steps"])
    s = MgritSolver(prob, TimeHierarchy.build(grid, mg["factors"]),
                    CycleSpec(kind="V", gamma=1, max_iters=50, spatial_strategy=mg["spatial_strategy"]),
                    StoppingCriterion(tolerance=mg["tolerance"]))
    torch.cuda.synchronize(); t2 = time.perf_counter()
    run, _ = s.solve(gather_solution=False)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    run, _ = s.solve(gather_solution=False)
    torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"rep {rep}: problem {t1-t0:.2f} setup {t2-t1:.2f} first solve {t3-t2:.2f} second solve {t4-t3:.2f} its {run.iterations}", flush=True)
    del s
    prob.close()
    torch.cuda.empty_cache()
