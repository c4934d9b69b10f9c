"""Break down the e2e leg of bench.py (dev tool)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import bench
from paper_1912_03106_b200 import (GpuFemProblem, MgritSolver, CycleSpec, StoppingCriterion,
                                   TimeHierarchy, build_uniform_grid, NullTransport)
spec = bench.headline_spec()
torch.cuda.init(); torch.zeros(1, device='cuda')
for rep in range(2):
    t = [time.perf_counter()]
    p = GpuFemProblem(spec, device=0); torch.cuda.synchronize(); t.append(time.perf_counter())
    grid = build_uniform_grid(0.0, spec["tf"], spec["n_steps"])
    mg = spec["mgrit"]
    s = MgritSolver(p, TimeHierarchy.build(grid, mg["factors"]),
                    CycleSpec(kind="V", gamma=1, spatial_strategy=mg["spatial_strategy"]),
                    StoppingCriterion(tolerance=1e-7), NullTransport()); torch.cuda.synchronize(); t.append(time.perf_counter())
    run, sol = s.solve(gather_solution=True); torch.cuda.synchronize(); t.append(time.perf_counter())
    h = sol.cpu(); t.append(time.perf_counter())
    hp = torch.empty(sol.shape, dtype=sol.dtype, pin_memory=True); hp.copy_(sol); torch.cuda.synchronize(); t.append(time.perf_counter())
    d = np.diff(t)
    print(f"rep {rep}: problem {d[0]:.3f}s solver-setup {d[1]:.3f}s solve+materialize {d[2]:.3f}s "
          f"D2H pageable {d[3]:.3f}s D2H pinned(+alloc) {d[4]:.3f}s  run.setup {run.setup_seconds:.3f} run.solve {run.solve_seconds:.3f}", flush=True)
    p.close()
