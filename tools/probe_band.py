"""Per-call timing of the banded-Cholesky Phi for the batch shapes of the
config-2 MGRIT solve (dev tool)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1912_03106_b200 import GpuFemProblem, configs, build
build.build()
if len(sys.argv) > 1 and sys.argv[1] == "cfg4":
    spec = configs.config4()
    shapes = [(0, 4096), (0, 1024), (0, 1), (1, 256), (1, 1)]
else:
    spec = configs.config2(N=128, n_steps=2 ** 14, levels=3, grids=2, strategy="delayed")
    shapes = [(0, 1024), (0, 64), (0, 1), (1, 64), (1, 1)]
if len(sys.argv) > 2:                      # only these "level:B" shapes
    shapes = [tuple(int(x) for x in a.split(":")) for a in sys.argv[2:]]
prob = GpuFemProblem(spec, inner="cholesky")
dev = prob.device
for level, B in shapes:
    n = prob.spatial.size(level)
    U = torch.as_tensor(np.random.default_rng(0).standard_normal((B, n)) * 1e-3, device=dev)
    dt = 0.02 / 2 ** 14
    inv = torch.full((B,), 1.0 / dt, dtype=torch.float64, device=dev)
    src = torch.as_tensor(prob.source_values(np.full(B, 0.01)), device=dev)
    out = torch.empty_like(U)
    prob.phi_batch(level, U, inv, src, out)        # factor
    torch.cuda.synchronize()
    reps = 20 if B * n < 1e8 else 3
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        prob.phi_batch(level, U, inv, src, out)
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / reps
    prob.profile(True)
    prob.phi_batch(level, U, inv, src, out)
    torch.cuda.synchronize()
    pr = prob.profile_read(reset=True)
    prob.profile(False)
    print(f"level {level} n={n} B={B}: {e0.elapsed_time(e1)/reps*1e3:.0f} us/call (gpu), "
          f"{wall*1e6:.0f} us/call (wall), band kernels {pr[2]['total_ms']*1e3:.0f} us", flush=True)
