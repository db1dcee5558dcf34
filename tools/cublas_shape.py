"""cuBLAS DGEMM on the layer-step shape: 256 independent (256 x 512) @ (512 x 512)^T products."""
import torch

for (T, M, N, K) in [(256, 256, 512, 512), (64, 256, 512, 512), (1, 256, 512, 512), (64, 16, 512, 512)]:
    a = torch.randn(T, M, K, dtype=torch.float64, device="cuda")
    b = torch.randn(T, N, K, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.bmm(a, b.transpose(1, 2))
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        torch.bmm(a, b.transpose(1, 2))
    e.record()
    e.synchronize()
    ms = s.elapsed_time(e) / 10
    print(f"bmm T={T} M={M} N={N} K={K}: {ms*1e3:.1f} us  {2*T*M*N*K/(ms*1e-3)/1e12:.2f} TF/s")
