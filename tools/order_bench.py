"""Bench of the injection-order search on planner-derived
op-cost tables: N synthetic mini-batches are planned on the device
(pp_plan_grid), their micro-batches priced (OpCostTable::from_shapes on the
device), then pp_order_search_device picks every mini-batch's injection order
(order_microbatches with plan_iteration's simulate evaluator).  Reports
orders/s (device, CUDA events, tables resident) and the reference's
order_microbatches on the host cores over a bounded sample.

    python tools/order_bench.py [--config C1] [--n 1024] [--clusters 3]"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def tables(planner, cfg, n_mb):
    from paper_2311_10418_b200 import capi
    from paper_2311_10418_b200 import workloads as W
    grid, model = W.grid(), W.model(cfg)
    s = W.dataset(cfg, n_mb)
    off = W.seg_offsets(cfg, n_mb)
    res = planner.plan_batch(s, off, grid, model, cfg.stages, 1, cfg.mem_cap, cfg.interval)
    shapes, mb_off = [], [0]
    for q in range(n_mb):
        ordered = res["ordered"][off[q]:off[q + 1]]
        a = 0
        for e in res["splits"][off[q]:off[q] + res["count"][q]]:
            blk = ordered[a:e]
            shapes.append((e - a, max(0, blk[:, 1].max()), max(0, blk[:, 2].max())))
            a = e
        mb_off.append(len(shapes))
    tf, tb, act = planner.op_costs(np.array(shapes, np.int64), grid, model)
    return tf, tb, act, np.array(mb_off, np.int64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--clusters", type=int, default=3)
    ap.add_argument("--limit-mult", type=float, default=2.5)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--ref-sample", type=int, default=64)
    args = ap.parse_args()
    import torch
    from oracle.bind import Reference, reference_available
    from paper_2311_10418_b200 import capi
    from paper_2311_10418_b200 import workloads as W
    cfg = W.CONFIGS[args.config]
    planner = capi.Planner(0)
    tf, tb, act, mb_off = tables(planner, cfg, args.n)
    C = tf.shape[1]
    lim = np.full(C, args.limit_mult * act.max())
    dev = torch.device("cuda:0")
    d_in = [torch.from_numpy(x).to(dev) for x in (tf, tb, act)]
    d_off = torch.from_numpy(mb_off).to(dev)
    S = args.n
    d = {"order": torch.empty(len(tf), dtype=torch.int32, device=dev),
         "makespan": torch.empty(S, dtype=torch.float64, device=dev),
         "bubble_ratio": torch.empty(S, dtype=torch.float64, device=dev),
         "deadlock": torch.empty(S, dtype=torch.int32, device=dev),
         "device_stats": torch.empty((S, C, 5), dtype=torch.float64, device=dev),
         "status": torch.empty(S, dtype=torch.int32, device=dev)}
    planner.order_search_device(*d_in, d_off, mb_off, lim, d, args.clusters, 0.0)  # warm-up
    st = torch.cuda.current_stream()
    planner.set_stream(st.cuda_stream)
    times = []
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        planner.order_search_device(*d_in, d_off, mb_off, lim, d, args.clusters, 0.0)
        e1.record(st)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    dev_s = float(np.median(times))
    got = {k: v.cpu().numpy() for k, v in d.items()}
    line = {"metric": "injection orders/s (order_microbatches + simulate evaluator)",
            "config": cfg.name, "minibatches": S, "micro_batches": int(len(tf)),
            "mean_microbatches_per_minibatch": float(len(tf) / S), "stages": C,
            "n_clusters": args.clusters, "permutations_per_minibatch": math.factorial(args.clusters),
            "device_s": dev_s, "device_orders_per_s": S / dev_s, "status_ok": int((got["status"] == 0).sum())}
    if reference_available():
        R = Reference()
        k = min(args.ref_sample, S)
        sub = mb_off[:k + 1]
        cores = os.cpu_count() or 1
        secs, exp = R.order_search(tf[:sub[-1]], tb[:sub[-1]], act[:sub[-1]], sub, lim, args.clusters, 0.0,
                                   threads=cores)
        same = bool(np.array_equal(exp["order"], got["order"][:sub[-1]]) and
                    exp["makespan"].tobytes() == got["makespan"][:k].tobytes())
        line["cpu_baseline"] = {"value": k / secs, "unit": "orders/s", "cores": cores, "kind": "reference",
                                "sample": f"first {k} mini-batches, one per std::thread", "wall_s": secs}
        line["parity_on_sample"] = same
        line["speedup_vs_cpu"] = (S / dev_s) / (k / secs)
    print(json.dumps(line), flush=True)
    planner.close()


if __name__ == "__main__":
    main()
