"""Per-call cost of level-0 batched Phi at the per-rank batch sizes of a
strong-scaling run (config 2: 1024 intervals / N ranks), with the real
per-interval 1/dt pattern of an F-offset (distinct rounding-level dt values,
so the factor grouping matches the solve) (dev tool)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1912_03106_b200 import GpuFemProblem, configs, build, build_uniform_grid
build.build()
spec = configs.config2(N=128, n_steps=2 ** 14, levels=3, grids=2, strategy="delayed")
prob = GpuFemProblem(spec, inner="cholesky")
dev = prob.device
grid = build_uniform_grid(0.0, spec["tf"], 2 ** 14).points
n = prob.spatial.size(0)
for B in [int(x) for x in (sys.argv[1:] or ["1024", "512", "256", "128", "64"])]:
    k = 5                                   # an F-offset inside every interval
    idx = 16 * np.arange(B) + k
    tp, tn = grid[idx], grid[idx + 1]
    inv = torch.as_tensor(1.0 / (tn - tp), device=dev)
    U = torch.as_tensor(np.random.default_rng(0).standard_normal((B, n)) * 1e-3, device=dev)
    src = torch.as_tensor(prob.source_values(tn), device=dev)
    out = torch.empty_like(U)
    prob.phi_batch(0, U, inv, src, out)              # factors / spikes
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        prob.phi_batch(0, U, inv, src, out)
    e1.record()
    torch.cuda.synchronize()
    ng = len(set((1.0 / (tn - tp)).tolist()))
    print(f"B={B:5d} ({ng} distinct dt): {e0.elapsed_time(e1) / reps * 1e3:8.0f} us/call", flush=True)
