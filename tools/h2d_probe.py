"""Pinned host -> device copy bandwidth on this box (context for bench.py's e2e)."""
import torch

n = 3 * 1024 ** 3 // 2
h = torch.empty(n, dtype=torch.bfloat16).pin_memory()
d = torch.empty(n, dtype=torch.bfloat16, device="cuda")
for chunks in (1, 4, 16):
    for _ in range(2):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        for c in range(chunks):
            s = slice(c * n // chunks, (c + 1) * n // chunks)
            d[s].copy_(h[s], non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"H2D {chunks} chunk(s): {n * 2 / ms / 1e6:.1f} GB/s")
