"""Where does the host-buffer (e2e) planning time go?  Times, for one C3
step of M mini-batches: the device-resident call, the host-buffer call, and
the bare pinned copies of the same bytes (development tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_10418_b200 import capi  # noqa: E402
from paper_2311_10418_b200 import workloads as W  # noqa: E402


def main(M=888, streams=3, reps=5, host_chunks=0):
    cfg = W.CONFIGS["C3"]
    s = W.dataset(cfg, M)
    off = W.seg_offsets(cfg, M)
    n = len(s)
    p = capi.Planner(0)
    p.set_tuning(streams=streams, host_chunks=host_chunks)
    print(f"streams {streams} host_chunks {host_chunks}")
    grid, model = W.grid(), W.model(cfg)
    pin = torch.from_numpy(s).pin_memory()
    pinned = []

    def alloc(shape, dtype):
        t = torch.empty(shape, dtype={np.int64: torch.int64, np.int32: torch.int32,
                                      np.float64: torch.float64}[dtype]).pin_memory()
        pinned.append(t)
        return t.numpy()

    out = capi.Planner.plan_buffers(n, M, alloc, order_only=True)
    args = (grid, model, cfg.stages, 1, cfg.mem_cap, cfg.interval)
    p.plan_batch(pin.numpy(), off, *args, out=out)
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        p.plan_batch(pin.numpy(), off, *args, out=out)
        t.append(time.perf_counter() - t0)
    print(f"host call      : {min(t) * 1e3:8.2f} ms  ({M / min(t):.0f} plans/s)")
    # the same call reading back only the per-plan scalars (no per-sample arrays)
    small = {k: (None if k in ("order", "ordered", "splits", "mb_times") else v) for k, v in out.items()}
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        p.plan_batch(pin.numpy(), off, *args, out=small)
        t.append(time.perf_counter() - t0)
    print(f"host, scalars  : {min(t) * 1e3:8.2f} ms  ({M / min(t):.0f} plans/s)")
    d_s = pin.cuda()
    d_off = torch.from_numpy(off).cuda()
    d_out = {k: torch.empty(v.shape, dtype=torch.from_numpy(v).dtype, device="cuda")
             for k, v in out.items() if v is not None}
    p.plan_batch_device(d_s, d_off, off, d_out, *args)
    torch.cuda.synchronize()
    t = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        p.plan_batch_device(d_s, d_off, off, d_out, *args)
        torch.cuda.synchronize()
        t.append(time.perf_counter() - t0)
    print(f"device call    : {min(t) * 1e3:8.2f} ms  ({M / min(t):.0f} plans/s)")
    h2d = pin.numel() * 8
    d2h = sum(v.nbytes for v in out.values() if v is not None)
    dst = torch.empty_like(pin, device="cuda")
    src = torch.empty(d2h // 8, dtype=torch.int64, device="cuda")
    back = torch.empty(d2h // 8, dtype=torch.int64).pin_memory()
    for name, fn in (("h2d copy", lambda: dst.copy_(pin, non_blocking=True)),
                     ("d2h copy", lambda: back.copy_(src, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / reps
        nb = h2d if name == "h2d copy" else d2h
        print(f"{name:15s}: {dt * 1e3:8.2f} ms  ({nb / dt / 1e9:.1f} GB/s, {nb / 1e6:.0f} MB)")
    st = p.stats()
    print("stats ms_total", round(st["ms_total"], 2), "kernel ms", [round(x, 2) for x in st["ms_kernel"]])


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
