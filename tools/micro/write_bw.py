"""HBM write-only and copy bandwidth on this GPU (torch fill_ / copy_ of a 4.29 GB
int32 buffer = the K29 output arrays' 8n bytes), CUDA events, best of 10."""
import torch

n = 1 << 30   # 4.29 GB of int32 = 8 bytes per K29 vertex
x = torch.empty(n, dtype=torch.int32, device="cuda")
y = torch.empty(n, dtype=torch.int32, device="cuda")
for name, fn, bytes_ in (("write (fill_)", lambda: x.fill_(-1), 4 * n),
                         ("copy (read+write)", lambda: y.copy_(x), 8 * n)):
    best = 1e9
    for _ in range(12):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{name}: {bytes_ / 1e9:.2f} GB in {best:.3f} ms = {bytes_ / best / 1e6:.0f} GB/s")
