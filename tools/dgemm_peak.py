"""cuBLAS DGEMM throughput via torch.matmul(float64): FP64 library reference peak."""
import json
import torch

out = {}
for n in (2048, 4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); torch.matmul(a, b); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out[f"dgemm_{n}_tflops"] = round(2 * n ** 3 / (best * 1e-3) / 1e12, 2)
print(json.dumps(out))
