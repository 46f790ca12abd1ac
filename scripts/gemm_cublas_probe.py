import torch, time
n, m, p = 4000000, 171, 81
V = torch.randn(m, n, dtype=torch.float64, device="cuda")   # rows = basis columns (column-major V)
Y = torch.randn(p, m, dtype=torch.float64, device="cuda")
for _ in range(3): Z = Y @ V
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): Z = Y @ V
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("cuBLAS fp64 GEMM (81 x 171) x (171 x 4M):", ms, "ms", 2*n*m*p/ms/1e9, "TFLOP/s")
