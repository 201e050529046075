"""A/B timing of planner tunings on a BASELINE config (development tool).

    python tools/ab_bench.py C3 296 "dp_pricing=1" "dp_pricing=0" "dp_pricing=0,compact_band=1"
Each variant: one-stream planning of M mini-batches, best of 3, per-kernel
device ms (CUDA events) from pp_stats."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_10418_b200 import capi  # noqa: E402
from paper_2311_10418_b200 import workloads as W  # noqa: E402


def main():
    name, M = sys.argv[1], int(sys.argv[2])
    cfg = W.CONFIGS[name]
    s = W.dataset(cfg, M)
    off = W.seg_offsets(cfg, M)
    ref = None
    for spec in sys.argv[3:]:
        kv = dict(x.split("=") for x in spec.split(",") if x)
        streams = int(kv.pop("streams", 1))
        tune = {k: bool(int(v)) for k, v in kv.items()}
        p = capi.Planner(0)
        p.set_tuning(streams=streams, **tune)
        r = p.plan_batch(s, off, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
        best, bst = 1e9, None
        for _ in range(3):
            t0 = time.perf_counter()
            r = p.plan_batch(s, off, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
            dt = time.perf_counter() - t0
            if dt < best:
                best, bst = dt, p.stats()
        sig = (r["t_max_used"].tobytes(), r["objective"].tobytes(), r["count"].tobytes())
        same = "ref" if ref is None else ("same" if sig == ref else "DIFFERENT")
        ref = ref or sig
        ks = {nm.split(" (")[0]: round(v, 3) for nm, v in zip(capi.KERNEL_NAMES, bst["ms_kernel"]) if v > 0}
        print(f"{name} M={M} [{spec}] {best * 1e3:.2f} ms wall, {M / best:.0f} plans/s, {same}; kernels ms {ks}; "
              f"band MB {bst['band_bytes'] / 1e6:.0f}", flush=True)
        p.close()


if __name__ == "__main__":
    main()
