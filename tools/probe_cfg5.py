"""Quick cfg5 probe: batched Phi timing on the 256^2 mesh (dev tool)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1912_03106_b200 import GpuFemProblem, configs, build
build.build()
spec = configs.config5()
prob = GpuFemProblem(spec, rtol=1e-10)
n = prob.spatial.size(0)
dev = prob.device
for B in [int(a) for a in (sys.argv[1:] or [64, 256, 1024])]:
    U = torch.as_tensor(np.random.default_rng(0).standard_normal((B, n)), device=dev)
    inv = torch.full((B,), 1.0 / spec['dt'], dtype=torch.float64, device=dev)
    src = torch.zeros(B, 0, dtype=torch.float64, device=dev)
    out = torch.empty_like(U)
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        prob.phi_batch(0, U, inv, src, out)
        st = prob.last_stats()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    bytes_ = st['column_iters'] * 64 * n * 8 / 8 + B * 40 * n
    print(f"B={B} n={n} time={dt*1e3:.1f} ms batch_iters={st['batch_iters']} col_iters={st['column_iters']} "
          f"launches={st['launches']} stepDOF/s={B*n/dt:.3e} GB/s(64n model)={(st['column_iters']*64*n + B*40*n)/dt/1e9:.0f}", flush=True)
