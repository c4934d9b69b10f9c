"""dev: determinism / A-B of the band chain kernels (one Phi batch, run several times)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1912_03106_b200 import GpuFemProblem, configs, build
N = int(sys.argv[1]); B = int(sys.argv[2]); nf = int(sys.argv[3]) if len(sys.argv) > 3 else 2
REPS = int(os.environ.get('DBG_REPS', '4'))
spec = configs.config4(N=N)
spec["n_spatial_grids"] = 1
prob = GpuFemProblem(spec, inner="cholesky")
prob2 = GpuFemProblem(spec, inner="cholesky") if os.environ.get('DBG_TWO') else None
n = prob.spatial.size(0)
rng = np.random.default_rng(5)
U = rng.standard_normal((B, n)) * 1e-3
dt0 = 0.02 / 2 ** 16
mult = 1 + rng.integers(0, nf, B)
tn = np.sort(rng.uniform(0.001, 0.02, B))
tp = tn - dt0 * mult
dev = prob.device
Ud = torch.as_tensor(U, device=dev)
inv = torch.as_tensor(1.0 / (tn - tp), device=dev)
src = torch.as_tensor(prob.source_values(tn), device=dev)
outs = []
for r in range(REPS):
    out = torch.empty(B, n, dtype=torch.float64, device=dev)
    prob.phi_batch(0, Ud, inv, src, out)
    outs.append(out.cpu().numpy())
ref = outs[0]
if prob2 is not None:
    o2 = torch.empty(B, n, dtype=torch.float64, device=dev)
    prob2.phi_batch(0, Ud, inv, src, o2)
    d = np.abs(o2.cpu().numpy() - ref).max(axis=1) / np.abs(ref).max(axis=1)
    print(f"second problem (fresh factors/spikes): max rel diff {d.max():.3e}")
for r in range(1, REPS):
    d = np.abs(outs[r] - ref).max(axis=1) / np.abs(ref).max(axis=1)
    print(f"N={N} B={B} rep {r}: max rel diff {d.max():.3e}, bad cols {np.nonzero(d > 1e-14)[0][:20]}")
import scipy.sparse.linalg as spla
from oracle import fem2d
lv = fem2d.make_problem(spec).levels[0]
dts = tn - tp
F = np.stack([fem2d.make_problem(spec).forcing(float(t)) for t in tn]) if B <= 200 else None
refp = fem2d.make_problem(spec)
exp = np.empty_like(U)
for dt in np.unique(dts):
    idx = np.nonzero(dts == dt)[0]
    lu = spla.splu((lv.K + lv.M * (1.0 / dt)).tocsc())
    Fi = np.stack([refp.forcing(float(t)) for t in tn[idx]])
    exp[idx] = lu.solve((Fi + (1.0 / dt) * (lv.M @ U[idx].T).T).T).T
for r in range(REPS):
    err = np.linalg.norm(outs[r] - exp, axis=1) / np.linalg.norm(exp, axis=1)
    bad = np.nonzero(err > 1e-11)[0]
    print(f"  rep {r}: max err {err.max():.3e}, bad cols {bad[:40]} ({len(bad)})")
