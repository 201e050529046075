"""Pinned host<->device copy bandwidth on this box (development probe)."""
import time
import torch
for mb in (116, 175):
    n = mb * 1024 * 1024 // 8
    h = torch.empty(n, dtype=torch.float64).pin_memory()
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    for direction in ("h2d", "d2h"):
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        print(f"{direction} {mb} MB: {mb / 1024 / dt:.1f} GB/s ({dt * 1e3:.2f} ms)")
