"""cuBLAS DGEMM ceiling (torch.matmul float64, 8192^3), the library FP64 roofline reference."""
import json
import torch

n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(2):
    torch.matmul(a, b)
torch.cuda.synchronize()
best = 0.0
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    best = max(best, 2 * n**3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
print(json.dumps({"cublas_dgemm_tflops_8192": round(best, 3)}))
