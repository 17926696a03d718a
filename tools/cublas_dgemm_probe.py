"""Run one cuBLAS DGEMM at the cfg4 update shape (for an ncu capture)."""
import torch
M, N = 1 << 20, 1024
A = torch.randn(M, N, dtype=torch.float64, device="cuda")
B = torch.randn(N, N, dtype=torch.float64, device="cuda")
C = torch.empty(M, N, dtype=torch.float64, device="cuda")
for _ in range(2):
    torch.matmul(A, B, out=C)
torch.cuda.synchronize()
print("ok")
