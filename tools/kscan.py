"""GEMM time vs k at m = n = 16384, N = 14 (CUDA events): the k-independent part
is the per-(tile, modulus) epilogue cost that short-K products cannot hide."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_08009_b200 import oz2
from paper_2504_08009_b200.inputs import phi_matrix_torch, SEED_A, SEED_B
n = 16384
for k in (256, 1024, 4096, 16384):
    A = phi_matrix_torch(n, k, 1.0, SEED_A, device="cuda")
    B = phi_matrix_torch(k, n, 1.0, SEED_B, device="cuda")
    C = oz2.dgemm(A, B, 14)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        oz2.dgemm(A, B, 14, out=C)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 3
    print(f"k={k}: {t:.2f} ms, {2 * n * n * k / t / 1e9:.1f} TFLOPS")
