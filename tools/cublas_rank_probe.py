"""Reference ceiling for the inversion's trailing update: cuBLAS batched DGEMM C += A W with
C (B x n x n), A (B x n x k), W (B x k x n) -- the same traffic shape as a rank-k pass -- timed
with CUDA events.  python tools/cublas_rank_probe.py [n=512] [B=512]"""
import sys
import torch
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
B = int(sys.argv[2]) if len(sys.argv) > 2 else 512
C = torch.randn(B, n, n, dtype=torch.float64, device="cuda")
for k in (32, 64, 128, 256):
    A = torch.randn(B, n, k, dtype=torch.float64, device="cuda")
    W = torch.randn(B, k, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        C.baddbmm_(A, W)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        C.baddbmm_(A, W)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    tf = 2.0 * B * n * n * k / (ms * 1e-3) / 1e12
    print(f"n {n} B {B} k {k}: {ms:.3f} ms  {tf:.2f} TFLOP/s ({100 * tf / 36.945:.1f}% of DMMA peak)")
