"""Per-(level, batch) time breakdown of the batched Phi calls inside one
config-2/3/4 MGRIT solve (dev tool; CUDA events around every call)."""
import collections, json, sys, time
import torch
sys.path.insert(0, '.')
from paper_1912_03106_b200 import (GpuFemProblem, CycleSpec, StoppingCriterion, TimeHierarchy,
                                   build_uniform_grid, MgritSolver, configs, build)
build.build()
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
if name == "cfg2":
    spec = configs.config2(grids=2, strategy="delayed")
elif name == "cfg3":
    spec = configs.config3(grids=2, strategy="delayed")
elif name == "cfg4":
    spec = configs.config4(grids=2, strategy="delayed")
elif name == "cfg4s":
    spec = configs.config2(N=128, n_steps=2 ** 14, levels=4, grids=2, strategy="delayed")
else:
    raise SystemExit(name)
if "merge" in sys.argv[2:]:
    spec["inner"]["dt_merge_rtol"] = 1e-12
prob = GpuFemProblem(spec)
mg = spec["mgrit"]
grid = build_uniform_grid(0.0, spec["tf"], spec["n_steps"])


def make():
    return MgritSolver(prob, TimeHierarchy.build(grid, mg["factors"]),
                       CycleSpec(kind="V", gamma=1, max_iters=50,
                                 spatial_strategy=mg["spatial_strategy"]),
                       StoppingCriterion(tolerance=mg["tolerance"]))


make().solve(gather_solution=False)          # warm (factors cached)
torch.cuda.synchronize()
rec = []
orig = prob.phi_batch


def timed(level, U, *a, **k):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = orig(level, U, *a, **k)
    e1.record()
    rec.append((level, U.shape[0], e0, e1))
    return r


import inspect
timed.__signature__ = inspect.signature(orig)
prob.phi_batch = timed
t0 = time.perf_counter()
run, _ = make().solve(gather_solution=False)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
agg = collections.defaultdict(lambda: [0, 0.0])
for lv, B, e0, e1 in rec:
    a = agg[(lv, B)]
    a[0] += 1
    a[1] += e0.elapsed_time(e1)
tot = sum(v[1] for v in agg.values())
print(json.dumps({"wall_s": wall, "iterations": run.iterations, "phi_ms": tot,
                  "history": [run.initial_residual] + run.residual_norms}))
for k in sorted(agg, key=lambda k: -agg[k][1]):
    n, ms = agg[k]
    print(f"grid {k[0]} B={k[1]:5d}: {n:5d} calls, {ms:8.1f} ms, {ms / n * 1e3:7.0f} us/call")
free, total = torch.cuda.mem_get_info()
print(f"GPU memory in use {(total - free) / 1e9:.1f} GB of {total / 1e9:.1f} GB")
