"""e2e setup in the bench's order: a first problem solved 5 times and kept
alive, then a second problem + solver built and timed (dev tool;
PG_DEBUG_SETUP=1 prints the band_factors host/kernel split)."""
import os, sys, time
import torch
sys.path.insert(0, '.')
import bench
from paper_1912_03106_b200 import (GpuFemProblem, MgritSolver, CycleSpec, StoppingCriterion,
                                   TimeHierarchy, build_uniform_grid, NullTransport)
spec = bench.headline_spec()
grid = build_uniform_grid(0.0, spec["tf"], spec["n_steps"])
mg = spec["mgrit"]


def make(p):
    return MgritSolver(p, TimeHierarchy.build(grid, mg["factors"]),
                       CycleSpec(kind="V", gamma=1, spatial_strategy=mg["spatial_strategy"]),
                       StoppingCriterion(tolerance=1e-7), NullTransport())


p1 = GpuFemProblem(spec, device=0)
s1 = make(p1)
for _ in range(5):
    s1.solve(gather_solution=False)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    p2 = GpuFemProblem(spec, device=0)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    s2 = make(p2)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"rep {rep}: problem {t1 - t0:.3f} s, solver setup {t2 - t1:.3f} s", file=sys.stderr, flush=True)
    del s2
    p2.close()
