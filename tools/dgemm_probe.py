import torch
x = torch.randn(4096, 4096, dtype=torch.float64, device="cuda")
for _ in range(3):
    y = torch.matmul(x, x)
torch.cuda.synchronize()
