"""Pinned host<->device copy bandwidth on this box (context for the e2e number)."""
import torch

for mb in (64, 256, 1024):
    n = mb * 2 ** 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    d.copy_(h, non_blocking=True)
    e1.record()
    h.copy_(d, non_blocking=True)
    e2.record()
    torch.cuda.synchronize()
    print(f"{mb} MiB: H2D {n / e0.elapsed_time(e1) / 1e6:.1f} GB/s, D2H {n / e1.elapsed_time(e2) / 1e6:.1f} GB/s")
