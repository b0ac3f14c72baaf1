import torch, numpy as np, time, sys
sys.path.insert(0, '.')
from paper_2504_08009_b200 import oz2
from paper_2504_08009_b200.inputs import phi_matrix_torch, SEED_A, SEED_B
n = 16384
A = phi_matrix_torch(n, n, 1.0, SEED_A, device="cuda"); B = phi_matrix_torch(n, n, 1.0, SEED_B, device="cuda")
Cd = oz2.dgemm(A, B, 14)
Ah = torch.empty((n, n), dtype=torch.float64, pin_memory=True); Ah.copy_(A)
Bh = torch.empty((n, n), dtype=torch.float64, pin_memory=True); Bh.copy_(B)
Ch = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
oz2.dgemm_host(Ah.numpy(), Bh.numpy(), 14, out=Ch.numpy())
assert torch.equal(Ch.cuda().view(torch.int64), Cd.view(torch.int64)), "host path differs"
for i in range(3):
    t = time.perf_counter(); oz2.dgemm_host(Ah.numpy(), Bh.numpy(), 14, out=Ch.numpy()); dt = time.perf_counter() - t
    print(f"e2e {dt*1e3:.1f} ms  {2*n**3/dt/1e12:.1f} TFLOPS")
# raw copy bandwidths (pinned host <-> device), for the e2e bound
for name, src, dst in (("H2D", Ah, A), ("D2H", Cd, Ch)):
    torch.cuda.synchronize(); t = time.perf_counter()
    dst.copy_(src, non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"{name} {src.numel() * 8 / dt / 1e9:.1f} GB/s ({dt*1e3:.1f} ms for 2.15 GB)")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t = time.perf_counter()
with torch.cuda.stream(s1): A.copy_(Ah, non_blocking=True)
with torch.cuda.stream(s2): Ch.copy_(Cd, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"H2D+D2H concurrent: {dt*1e3:.1f} ms for 2 x 2.15 GB")
