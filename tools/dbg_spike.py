"""dev: determinism of the SPIKE responses G (two fresh problems, same batch)."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1912_03106_b200 import GpuFemProblem, configs
N = int(sys.argv[1]); B = int(sys.argv[2])
spec = configs.config4(N=N)
spec["n_spatial_grids"] = 1
Gs = []
for rep in range(2):
    prob = GpuFemProblem(spec, inner="cholesky")
    n = prob.spatial.size(0)
    rng = np.random.default_rng(5)
    U = rng.standard_normal((B, n)) * 1e-3
    tn = np.sort(rng.uniform(0.001, 0.02, B))
    dev = prob.device
    inv = torch.full((B,), 2.0 ** 16 / 0.02, dtype=torch.float64, device=dev)
    out = torch.empty(B, n, dtype=torch.float64, device=dev)
    prob.phi_batch(0, torch.as_tensor(U, device=dev), inv,
                   torch.as_tensor(prob.source_values(tn), device=dev), out)
    torch.cuda.synchronize()
    lib = prob.lib
    lib.pg_dev_spike_g.argtypes = [ctypes.c_void_p] + [ctypes.c_int] * 4 + [ctypes.c_void_p]
    np_ = (n + 31) // 32 * 32
    got = {}
    for pi in range(3):
        for fwd in (1, 0):
            G = torch.zeros(512 * np_, dtype=torch.float64, device=dev)
            rc = lib.pg_dev_spike_g(prob.ctx, 0, pi, 0, fwd, ctypes.c_void_p(G.data_ptr()))
            if rc == 0:
                got[(pi, fwd)] = G.view(512, np_).cpu().numpy()
    Gs.append(got)
    print("rep", rep, "partitions with G:", sorted(got))
for key in Gs[0]:
    a, b = Gs[0][key], Gs[1][key]
    d = np.abs(a - b)
    rows = np.nonzero(d.max(axis=0) > 0)[0]
    cols = np.nonzero(d.max(axis=1) > 0)[0]
    print(key, "max diff", d.max(), "max |G|", np.abs(a).max(), "n bad rows", len(rows),
          "rows", rows[:10], "..", rows[-5:] if len(rows) else [], "blocks", np.unique(rows // 32)[:40],
          "cols", cols[:40], "n bad cols", len(cols))
