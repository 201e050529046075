"""Whole-epoch planning, device-resident from the dataset file to the
injection orders (every stage bit-exact with the reference, tests/):

  record-file bytes --pp_load_records_device--> samples (HBM)
  --pp_draw_minibatches_device--> token-budgeted mini-batches (run_plan's draw)
  --pp_plan_grid_device--> DP micro-batch plans (order_samples + make_slice_cost + dp_partition)
  --pp_plan_op_costs_device--> op-cost tables (OpCostTable::from_shapes)
  --pp_order_search_device--> injection orders + SimReport (order_microbatches + simulate)

Prints the time of each stage (CUDA events on the planner's stream) for a
C4-like epoch: GPT, 8 stages, ~2048 samples per mini-batch.

    python tools/epoch_pipeline.py [--n 4194304] [--budget 900000]"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096 * 1024)
    ap.add_argument("--budget", type=int, default=900_000)
    ap.add_argument("--stages", type=int, default=8)
    args = ap.parse_args()
    import torch
    from ingest_cases import random_file
    from paper_2311_10418_b200 import capi
    from paper_2311_10418_b200 import workloads as W
    data = random_file(args.n, seed=7, noise=False, max_len=8192)
    p = capi.Planner(0)
    st = torch.cuda.current_stream()
    p.set_stream(st.cuda_stream)
    p.set_tuning(streams=1)
    dev = torch.device("cuda:0")
    grid, model = W.grid(), capi.Model.uniform(args.stages, 2, False)
    C = args.stages

    def run():
        ev = []

        def mark():
            e = torch.cuda.Event(enable_timing=True)
            e.record(st)
            ev.append(e)

        pin = torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory()
        torch.cuda.synchronize()
        mark()
        d_bytes = pin.to(dev, non_blocking=True)
        mark()
        d_s = torch.empty((args.n + 8, 3), dtype=torch.int64, device=dev)
        n = p.load_records_device(d_bytes, len(data), 8192, d_s)
        mark()
        d_off = torch.empty(n + 1, dtype=torch.int64, device=dev)
        n_seg = p.draw_minibatches_device(d_s, n, args.budget, d_off)
        mark()
        h_off = d_off[:n_seg + 1].cpu().numpy()
        out = {"ordered": torch.empty((n, 3), dtype=torch.int64, device=dev),
               "splits": torch.empty(n, dtype=torch.int32, device=dev),
               "mb_times": torch.empty(n, dtype=torch.float64, device=dev),
               "count": torch.empty(n_seg, dtype=torch.int32, device=dev),
               "t_max_used": torch.empty(n_seg, dtype=torch.float64, device=dev),
               "objective": torch.empty(n_seg, dtype=torch.float64, device=dev),
               "status": torch.empty(n_seg, dtype=torch.int32, device=dev),
               "err_sample_id": torch.empty(n_seg, dtype=torch.int64, device=dev)}
        mark()
        p.plan_batch_device(d_s, d_off[:n_seg + 1], h_off, out, grid, model, C, 1, float("inf"), 5000.0)
        mark()
        d_tf, d_tb, d_act = (torch.empty(n * C, dtype=torch.float64, device=dev) for _ in range(3))
        mb_off = p.plan_op_costs_device(out["ordered"], d_off[:n_seg + 1], h_off, out["splits"], out["count"], grid,
                                        model, d_tf, d_tb, d_act)
        mark()
        n_mb = int(mb_off[-1])
        lim = np.full(C, 2.5 * float(d_act[:n_mb * C].max().item()))
        d_mbo = torch.from_numpy(mb_off).to(dev)
        o = {"order": torch.empty(n_mb, dtype=torch.int32, device=dev),
             "makespan": torch.empty(n_seg, dtype=torch.float64, device=dev),
             "bubble_ratio": torch.empty(n_seg, dtype=torch.float64, device=dev),
             "deadlock": torch.empty(n_seg, dtype=torch.int32, device=dev),
             "device_stats": None, "status": torch.empty(n_seg, dtype=torch.int32, device=dev)}
        mark()
        p.order_search_device(d_tf[:n_mb * C], d_tb[:n_mb * C], d_act[:n_mb * C], d_mbo, mb_off, lim, o, 3, 0.0)
        mark()
        torch.cuda.synchronize()

        return ev, n, n_seg, n_mb, out, o

    run()  # warm-up: module loads, scratch allocations
    ev, n, n_seg, n_mb, out, o = run()
    names = ["h2d file", "ingest", "draw", "(host: offsets, buffers)", "DP plans", "op costs",
             "(host: limits)", "order search"]
    ms = {k: ev[i].elapsed_time(ev[i + 1]) for i, k in enumerate(names)}
    line = {"metric": "whole-epoch planning, file -> injection orders (device)", "samples": n, "file_bytes": len(data),
            "minibatches": n_seg, "micro_batches": n_mb, "stages": C, "stage_ms": ms,
            "total_ms": ev[0].elapsed_time(ev[-1]),
            "plans_ok": int((out["status"] == 0).sum().item()), "orders_ok": int((o["status"] == 0).sum().item())}
    print(json.dumps(line), flush=True)
    p.close()


if __name__ == "__main__":
    main()
