"""Mid-size throughput probe (N = 14, m = n = k): CUDA-event time per oz2.dgemm call."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_08009_b200 import oz2
from paper_2504_08009_b200.inputs import phi_matrix_torch, SEED_A, SEED_B
for n in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2048,3072,4096,6144,8192").split(",")]:
    A = phi_matrix_torch(n, n, 1.0, SEED_A, device="cuda"); B = phi_matrix_torch(n, n, 1.0, SEED_B, device="cuda")
    C = oz2.dgemm(A, B, 14); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): oz2.dgemm(A, B, 14, out=C)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10
    print(f"{os.environ.get('OZ2_UP_TILES', 'default')} n={n}: {t:.3f} ms {2 * n**3 / t / 1e9:.1f} TFLOPS")
