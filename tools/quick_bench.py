"""Quick timing of the planner on the BASELINE configs (development tool)."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2311_10418_b200 import capi  # noqa: E402
from paper_2311_10418_b200 import workloads as W  # noqa: E402


def run(name, M, reps=3, first_wave=1, max_wave=16, streams=1):
    cfg = W.CONFIGS[name]
    s = W.dataset(cfg, M)
    off = W.seg_offsets(cfg, M)
    p = capi.Planner(0)
    # QB_TUNE="compact_band=0,band_trunc=0,slice_reuse=0": A/B switches
    tune = {k: bool(int(v)) for k, v in (kv.split("=") for kv in os.environ.get("QB_TUNE", "").split(",") if kv)}
    p.set_tuning(first_wave, max_wave, streams, **tune)
    r = p.plan_batch(s, off, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        r = p.plan_batch(s, off, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
        best = min(best, time.perf_counter() - t0)
    st = p.stats()
    print(f"{name} M={M}: {best*1e3:.2f} ms wall, {M/best:.2f} plans/s, status={set(r['status'].tolist())} "
          f"count0={r['count'][0]} t0={r['t_max_used'][0]} "
          f"stats={ {k: (round(v, 3) if isinstance(v, float) else v) for k, v in st.items()} }", flush=True)


if __name__ == "__main__":
    for spec in sys.argv[1:] or ["C1:1", "C1:64", "C2:1", "C2:16", "C3:1", "C3:8", "C4:64", "C4:512"]:
        n, m, *g = spec.split(":")
        run(n, int(m), streams=int(g[0]) if g else 1)
