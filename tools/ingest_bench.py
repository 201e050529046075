"""Bench of the dataset ingest: a record file of the
whole-epoch workload (C4: 4096 x 2048 = 8.39 M samples, FLANv2-like lognormal
lengths) parsed on the device (bytes resident in HBM, CUDA events), end to
end from pinned host bytes, and the mini-batch draw; next to the reference's
load_dataset (one host thread: it is a sequential ifstream parse) on the same
file from the page cache.

    python tools/ingest_bench.py [--n 8388608] [--reps 5]"""
import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096 * 2048)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--budget", type=int, default=65536)
    args = ap.parse_args()
    import torch
    from ingest_cases import random_file
    from oracle.bind import Reference, reference_available
    from paper_2311_10418_b200 import capi
    data = random_file(args.n, seed=7, noise=False)
    planner = capi.Planner(0)
    st = torch.cuda.current_stream()
    planner.set_stream(st.cuda_stream)
    d_bytes = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
    d_out = torch.empty((args.n + 16, 3), dtype=torch.int64, device="cuda")
    d_off = torch.empty(args.n + 17, dtype=torch.int64, device="cuda")
    n = planner.load_records_device(d_bytes, len(data), 8192, d_out)

    def timed(fn):
        ts = []
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(st)
            fn()
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        return float(np.median(ts))

    t_parse = timed(lambda: planner.load_records_device(d_bytes, len(data), 8192, d_out))
    n_seg = planner.draw_minibatches_device(d_out, n, args.budget, d_off)
    t_draw = timed(lambda: planner.draw_minibatches_device(d_out, n, args.budget, d_off))
    pin = torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory()
    out_pin = torch.empty((args.n + 16, 3), dtype=torch.int64).pin_memory()

    def e2e():
        d_bytes.copy_(pin, non_blocking=True)
        planner.load_records_device(d_bytes, len(data), 8192, d_out)
        out_pin[:n].copy_(d_out[:n], non_blocking=True)
    e2e()
    t_e2e = timed(e2e)
    # algorithmic bytes: the file read once, 24 B per sample written
    alg = len(data) + 24 * n
    line = {"metric": "dataset ingest (load_dataset over a record file)", "samples": n,
            "file_bytes": len(data), "device_s": t_parse, "device_GBps_file": len(data) / t_parse / 1e9,
            "device_samples_per_s": n / t_parse, "algorithmic_bytes": alg,
            "achieved_GBps_algorithmic": alg / t_parse / 1e9, "e2e_s": t_e2e,
            "e2e_samples_per_s": n / t_e2e, "draw_s": t_draw, "minibatches": n_seg,
            "token_budget": args.budget}
    peaks = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(peaks):
        pk = json.load(open(peaks))
        hbm = pk.get("hbm_gbs") or pk.get("hbm_GBps")
        if hbm:
            line["roofline"] = {"bound": "hbm", "peak": hbm, "frac": alg / t_parse / 1e9 / hbm}
    if reference_available():
        R = Reference()
        with tempfile.NamedTemporaryFile(suffix=".tsv", delete=False) as f:
            f.write(data)
            path = f.name
        R.load_record_file(path, 8192, cap=n + 1)  # page cache
        t0 = time.perf_counter()
        rc, ref, *_ = R.load_record_file(path, 8192, cap=n + 1)
        t_ref = time.perf_counter() - t0
        t0 = time.perf_counter()
        rc2, ref_off = R.draw_all(ref, args.budget)
        t_ref_draw = time.perf_counter() - t0
        got = d_out[:n].cpu().numpy()
        got_off = d_off[:n_seg + 1].cpu().numpy()
        line["cpu_baseline"] = {"value": n / t_ref, "unit": "samples/s", "cores": 1, "kind": "reference",
                                "sample": "the whole file, load_dataset(DatasetSpec{path}), page cache warm",
                                "wall_s": t_ref, "draw_wall_s": t_ref_draw}
        line["parity"] = bool(rc == 0 and np.array_equal(ref, got) and np.array_equal(ref_off, got_off))
        os.unlink(path)
    print(json.dumps(line), flush=True)
    planner.close()


if __name__ == "__main__":
    main()
