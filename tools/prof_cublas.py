"""cuBLAS DGEMM on the C2 Gaussian shapes (ncu comparator for gauss_kernel)."""
import torch
n, d = 16384, 512
A = torch.randn(n, n, dtype=torch.float64, device="cuda")
R = torch.randn(d, n, dtype=torch.float64, device="cuda")
for _ in range(2):
    S = A @ R.T
torch.cuda.synchronize()
