"""Strip solve vs natural-order band solve on the same inputs (dev tool).
usage: python tools/probe_strips.py [N] [B]"""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1912_03106_b200 import GpuFemProblem, configs, build
build.build()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
spec = configs.config2(N=N, n_steps=2 ** 14, levels=1)
spec["inner"]["dt_merge_rtol"] = 1e-12
prob = GpuFemProblem(spec, inner="cholesky")
dev = prob.device
n = prob.spatial.size(0)
rng = np.random.default_rng(0)
U = torch.as_tensor(rng.standard_normal((B, n)) * 1e-3, device=dev)
dt = 0.02 / 2 ** 14
inv_h = np.where(np.arange(B) % 5 == 0, 1.0 / (dt * (1 + 1e-9)), 1.0 / dt)
inv = torch.as_tensor(inv_h, device=dev)
src = torch.as_tensor(prob.source_values(np.linspace(0.001, 0.019, B)), device=dev)
G = torch.as_tensor(rng.standard_normal((3, n)), device=dev)
g_idx = torch.as_tensor((np.arange(B) % 4 - 1).clip(-1, 2).astype(np.int32), device=dev)
out = torch.empty_like(U)


def run(tag):
    prob.phi_batch(0, U, inv, src, out, g=G, g_idx=g_idx, inv_dt_host=inv_h)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        prob.phi_batch(0, U, inv, src, out, g=G, g_idx=g_idx, inv_dt_host=inv_h)
    e1.record()
    torch.cuda.synchronize()
    print(f"{tag}: {e0.elapsed_time(e1) / 3:.2f} ms per call", flush=True)
    return out.clone()


a = run("default")
prob.profile(True)
prob.phi_batch(0, U, inv, src, out, g=G, g_idx=g_idx, inv_dt_host=inv_h)
torch.cuda.synchronize()
print({k["name"]: round(k["total_ms"], 2) for k in prob.profile_read(reset=True) if k["launches"]})
prob.profile(False)
prob.close()
mode = os.environ.get("PG_STRIPS", "1")
sub = a[::max(1, B // 64)].cpu().numpy()
np.save(f"/tmp/strips_{N}_{mode}.npy", sub)
other = f"/tmp/strips_{N}_{'0' if mode != '0' else '1'}.npy"
if os.path.exists(other):
    o = np.load(other)
    rel = np.linalg.norm(sub - o, axis=1) / np.linalg.norm(o, axis=1)
    print(f"strips vs natural band solve, {len(rel)} sampled columns: max rel diff {rel.max():.3e}")
