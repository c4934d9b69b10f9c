"""Host-side profile of the e2e setup (problem + solver construction) (dev tool)."""
import cProfile, pstats, sys, time
import torch
sys.path.insert(0, '.')
import bench
from paper_1912_03106_b200 import (GpuFemProblem, MgritSolver, CycleSpec, StoppingCriterion,
                                   TimeHierarchy, build_uniform_grid, NullTransport)
spec = bench.headline_spec()
torch.zeros(1, device='cuda')


def setup():
    p = GpuFemProblem(spec, device=0)
    grid = build_uniform_grid(0.0, spec["tf"], spec["n_steps"])
    mg = spec["mgrit"]
    s = MgritSolver(p, TimeHierarchy.build(grid, mg["factors"]),
                    CycleSpec(kind="V", gamma=1, spatial_strategy=mg["spatial_strategy"]),
                    StoppingCriterion(tolerance=1e-7), NullTransport())
    torch.cuda.synchronize()
    return p, s


p, s = setup()
del s
p.close()
t0 = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
p, s = setup()
pr.disable()
print("setup", time.perf_counter() - t0)
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
