"""TRMM timing probe: oz2.trmm (K skipping) vs oz2.gemm on the masked matrix, CUDA events."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_08009_b200 import oz2
from paper_2504_08009_b200.inputs import phi_matrix_torch, SEED_A, SEED_B
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
A = phi_matrix_torch(n, n, 1.0, SEED_A, device="cuda")
B = phi_matrix_torch(n, n, 1.0, SEED_B, device="cuda")
T = A.tril()
Bw = B.clone()
def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
t1 = timed(lambda: oz2.trmm(A, Bw, 14, "L", "L"))
t2 = timed(lambda: oz2.gemm(T, B, 14))
print(f"{os.environ.get('OZ2_SYNC_KB', 'default')}: trmm {t1:.2f} ms, gemm(tri(A), B) {t2:.2f} ms")
