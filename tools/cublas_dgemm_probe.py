"""cuBLAS DGEMM (the roofline denominator) on this GPU, for an ncu capture of its kernel:
8192^3 and the c2 step shape as a strided batch (256 x (256x512)(512x512)^T)."""
import torch

a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
torch.matmul(a, b)
x = torch.randn(256, 256, 512, dtype=torch.float64, device="cuda")
w = torch.randn(256, 512, 512, dtype=torch.float64, device="cuda")
torch.bmm(x, w.transpose(1, 2))
torch.cuda.synchronize()
