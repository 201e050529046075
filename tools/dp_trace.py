"""Per-block phase timing of the DP kernel (development tool, GPU box).

    PP_TRACE=1 python -c "from paper_2311_10418_b200 import build as b; b.build()"   # here
    PIPEPLAN_B200_LIB=build/trace/libpipeplan_b200_trace.so python tools/dp_trace.py C3

Stamps (clock64, CTA 0 of the last DP launch): chain 0 start, 1 near tile
ready, 2 near-far + tile loads done, 3 triangle done, 4 states stored,
5 after the block barrier; worker 0: 8 start, 9 chunks done, 10 fold done.
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2311_10418_b200 import capi  # noqa: E402
from paper_2311_10418_b200 import workloads as W  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C3"
    cfg = W.CONFIGS[name]
    nblk = (cfg.n + 31) // 32
    buf = torch.zeros(nblk * 16, dtype=torch.int64, device="cuda")
    capi.lib.pp_debug_dp_trace.argtypes = [ctypes.c_void_p]
    assert capi.lib.pp_debug_dp_trace(ctypes.c_void_p(buf.data_ptr())) == 0
    # DP_FLAGS=1: the workers skip the far-far columns (wrong plans; isolates the chain's timing)
    assert capi.lib.pp_debug_dp_flags(int(os.environ.get("DP_FLAGS", "0"))) == 0
    p = capi.Planner(0)
    # QB_TUNE="slice_table=0": A/B switches, as in tools/quick_bench.py
    tune = {k: bool(int(v)) for k, v in (kv.split("=") for kv in os.environ.get("QB_TUNE", "").split(",") if kv)}
    p.set_tuning(**tune)
    M = int(os.environ.get("DP_M", "1"))  # mini-batches planned together (CTA 0 is traced)
    s = W.dataset(cfg, M)
    off = W.seg_offsets(cfg, M)
    for _ in range(2):
        p.plan_batch(s, off, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
    torch.cuda.synchronize()
    t = buf.view(nblk, 16).cpu().numpy().astype(np.int64)
    ok = t[:, 0] > 0
    t = t[ok]
    d = lambda a, b: t[:, b] - t[:, a]  # noqa: E731
    rows = [("chain: A prep (partials)", 0, 1), ("chain: unit wait", 1, 2),
            ("chain: triangle", 2, 3), ("chain: store states", 3, 4), ("chain: block barrier", 4, 5),
            ("worker0: far-far chunks", 8, 9), ("worker0: fold", 9, 10), ("worker0: to barrier", 10, 5),
            ("producer: wait for a free unit", 11, 12), ("producer: unit fill", 12, 13)]
    print(f"{name}: {len(t)} blocks traced; cycles per block (median / mean)")
    for lbl, a, b in rows:
        x = d(a, b)
        print(f"  {lbl:32s} {np.median(x):8.0f} {x.mean():8.0f}")
    per = np.diff(t[:, 0])
    print(f"  {'block period':32s} {np.median(per):8.0f} {per.mean():8.0f}")
    print(f"  total {t[-1, 5] - t[0, 0]} cycles")
    # the two halves per block: chain (partials, triangle, stores) vs worker 0
    # (far-far + its fold; blocks whose worker stamps were written)
    w_ok = (t[:, 8] > 0) & (t[:, 10] >= t[:, 8])
    ch = d(0, 4)
    wk = np.where(w_ok, t[:, 10] - t[:, 8], 0)
    print(f"  sum chain path {ch.sum()}  sum worker path {wk.sum()}  sum max {np.maximum(ch, wk).sum()}"
          f"  sum period {per.sum()}")
    q = max(1, len(t) // 8)
    print("  per eighth of the blocks (mean chain / worker / period):")
    for a in range(0, len(t), q):
        sl = slice(a, min(a + q, len(t)))
        pp = per[a:min(a + q, len(per))]
        print(f"    blocks {a:4d}+: {ch[sl].mean():7.0f} {wk[sl].mean():7.0f} {pp.mean() if len(pp) else 0:7.0f}")


if __name__ == "__main__":
    main()
