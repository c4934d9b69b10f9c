"""Bitwise A/B of the streamed PCG Phi between two library builds (dev tool):
python tools/probe_pcg_bits.py out.npy  (PINTGPU_LIB selects the build).
Mixed 1/dt batch: columns 0..B/2 share column 0's 1/dt (uniform fast path),
the rest differ."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1912_03106_b200 import GpuFemProblem, configs
spec = configs.config5()
prob = GpuFemProblem(spec, rtol=1e-10)
n = prob.spatial.size(0)
dev = prob.device
res = {}
for B, mixed in [(64, True), (256, False), (37, True)]:
    U = torch.as_tensor(np.random.default_rng(B).standard_normal((B, n)), device=dev)
    dt = np.full(B, spec['dt'])
    if mixed:
        dt[B // 2:] *= 1.0 + 1e-3 * np.arange(1, B - B // 2 + 1)
    inv = torch.as_tensor(1.0 / dt, device=dev)
    src = torch.zeros(B, 0, dtype=torch.float64, device=dev)
    out = torch.empty_like(U)
    prob.phi_batch(0, U, inv, src, out)
    st = prob.last_stats()
    o = out.cpu().numpy()
    res[f"{B}_sha"] = np.frombuffer(__import__("hashlib").sha256(o.tobytes()).digest(), np.uint8)
    res[f"{B}_sum"] = np.array([np.sum(np.abs(o))])
    res[f"{B}_iters"] = np.array([st['batch_iters'], st['column_iters']])
np.savez(sys.argv[1], **res)
print("saved", {k: v for k, v in res.items() if k.endswith('iters')})
