"""Bench of padding_vs_packing_report on the device:
the acceptance-suite setting scaled to a whole dataset (GPT, 4 stages,
token budget 65536, max_seq_lens 512 / 2048 / 8192) against the reference's
report (one host thread: it is a sequential loop) on a bounded sample.

    python tools/report_bench.py [--n 100000] [--iters 0] [--ref-iters 40]"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100_000)
    ap.add_argument("--iters", type=int, default=0)
    ap.add_argument("--ref-iters", type=int, default=40)
    ap.add_argument("--interval", type=float, default=500.0)
    args = ap.parse_args()
    from oracle.bind import Reference, reference_available
    from paper_2311_10418_b200 import capi
    from paper_2311_10418_b200 import workloads as W
    g, m = W.grid(), capi.Model.uniform(4, 2, False)
    s = capi.synthetic_dataset(args.n, 16384, 7, W.INPUT_DIST, None)
    lens = [512, 2048, 8192]
    p = capi.Planner(0)
    p.padding_report(s, lens, g, m, 65536, args.interval, max(1, args.ref_iters))  # warm-up
    t0 = time.perf_counter()
    rows = p.padding_report(s, lens, g, m, 65536, args.interval, args.iters)
    t = time.perf_counter() - t0
    n_mb = len(p.draw_minibatches(s, 65536)) - 1
    iters = n_mb if args.iters == 0 else min(args.iters, n_mb)
    line = {"metric": "padding_vs_packing_report iterations/s (3 methods x 3 max_seq_lens per mini-batch)",
            "samples": args.n, "minibatches": iters, "device_wall_s": t, "iterations_per_s": iters / t,
            "rows": [{k: (float(r[k]) if k != "method" else int(r[k])) for k in rows.dtype.names} for r in rows]}
    if reference_available():
        R = Reference()
        k = min(args.ref_iters, iters)
        secs, exp = R.padding_report(s, lens, g, m, 65536, args.interval, k)
        got = p.padding_report(s, lens, g, m, 65536, args.interval, k)
        line["cpu_baseline"] = {"value": k / secs, "unit": "iterations/s", "cores": 1, "kind": "reference",
                                "sample": f"first {k} mini-batches", "wall_s": secs}
        line["parity_on_sample"] = got.tobytes() == exp.tobytes()
    print(json.dumps(line), flush=True)
    p.close()


if __name__ == "__main__":
    main()
