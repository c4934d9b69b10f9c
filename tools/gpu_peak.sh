mkdir -p gpurun_out
./tools/fp64_peak > gpurun_out/fp64_peak.json 2>&1
python - >> gpurun_out/fp64_peak.json 2>&1 <<'PY'
import torch, json
for N in (4096, 8192):
    a = torch.randn(N, N, dtype=torch.float64, device='cuda'); b = torch.randn_like(a)
    for _ in range(2): c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    print(json.dumps({"kind": "cublas_dgemm", "N": N, "ms": best, "tflops": 2 * N**3 / best / 1e9}))
PY
