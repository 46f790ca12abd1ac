"""Random-gather ceiling vs streaming (diagnostic, SURVEY §8(d) metric 1)."""
import torch, json
dev = torch.device("cuda:0")
n, nnz = 4_000_000, 128_000_000
x = torch.randn(n, dtype=torch.float64, device=dev)
idx = torch.randint(0, n, (nnz,), device=dev, dtype=torch.int64)
idx32 = idx.to(torch.int32)
big = torch.empty(nnz // 2 * 3, dtype=torch.float64, device=dev)  # ~1.5 GB
dst = torch.empty_like(big)
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
g_ms = t(lambda: x[idx])
c_ms = t(lambda: dst.copy_(big))
print(json.dumps({"gather_128M_ms": g_ms, "gather_GBps_idx8+val8+out8": nnz * 24 / g_ms / 1e6,
                  "copy_1.5GB_ms": c_ms, "copy_GBps": 2 * big.numel() * 8 / c_ms / 1e6}))
