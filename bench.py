"""Benchmark: micro-batch plans/sec on 8192-sequence mini-batches (BASELINE.json
config C3: GPT cost model, 16 stages, binding activation-memory cap, 128-candidate
t_max sweep), at N GPUs of one node (weak scaling: every rank plans its own
M mini-batches per step, one final NCCL gather of the plans per step).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

A "step" = planning M independent mini-batches (order_samples(Sort) +
make_slice_cost + dp_partition each) through pp_plan_grid_device with the
inputs already resident in HBM; distinct mini-batches every step, and the
per-step band traffic (~21 MB per plan) exceeds L2.  `e2e` repeats the
measurement through the host-buffer C-ABI call pp_plan_grid (pinned samples in,
plans out).  `--impl reference` times the unmodified reference planner
(oracle/_ref) on the host cores with run_plan's worker-pool model.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "micro-batch plans/sec (8192-seq mini-batch, t_max sweep)"
UNIT = "plans/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for k, v in zip(names, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(k)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def traffic_record(config_name):
    """Latest profiles/r*/traffic_<config>.json (per-plan DRAM bytes per kernel
    from an ncu --set full capture), or None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", f"traffic_{config_name.lower()}.json")))
    if not files:
        return None
    with open(files[-1]) as f:
        return json.load(f)


def cpu_baseline_sample(cfg, threads, plans):
    """The unmodified reference (oracle/_ref) on the host cores: `plans`
    8192-seq mini-batches (one per thread) through order_samples +
    make_slice_cost + dp_partition in run_plan's worker pool."""
    from oracle.bind import Reference, reference_available
    from paper_2311_10418_b200 import workloads as W

    if not reference_available():
        return None
    ref = Reference()
    s = W.dataset(cfg, plans)
    off = W.seg_offsets(cfg, plans)
    secs, tm, ob, cnt, st = ref.plan_batch_timed(s, off, W.grid(), W.model(cfg), cfg.stages, 1,
                                                 cfg.mem_cap, cfg.interval, threads)
    return {"value": plans / secs, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{plans} x {cfg.n}-seq mini-batches of {cfg.name}, one per std::thread "
                      f"(run_plan pool), wall {secs:.1f} s",
            "t_max_first": float(tm[0]), "status_ok": int((st == 0).sum())}


def run_reference(args, rank, world):
    """--impl reference: rank 0 times the reference CPU planner; others exit."""
    if rank != 0:
        return
    from paper_2311_10418_b200 import workloads as W

    cfg = W.CONFIGS[args.config]
    cores = os.cpu_count() or 1
    from oracle.bind import Reference, reference_available

    if not reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    ref = Reference()
    # warm-up steps: bounded C1 plans through the same code path (page-in)
    c1 = W.CONFIGS["C1"]
    s1 = W.dataset(c1, max(args.warmup, 1))
    ref.plan_batch_timed(s1, W.seg_offsets(c1, max(args.warmup, 1)), W.grid(), W.model(c1), c1.stages,
                         1, c1.mem_cap, c1.interval, min(cores, max(args.warmup, 1)))
    # timed: max(K, cores) 8192-seq mini-batches, one per std::thread of
    # run_plan's pool over ALL host cores (a mini-batch is one step's unit)
    K = args.steps
    P = max(K, cores)
    s = W.dataset(cfg, P)
    secs, tm, ob, cnt, st = ref.plan_batch_timed(s, W.seg_offsets(cfg, P), W.grid(), W.model(cfg),
                                                 cfg.stages, 1, cfg.mem_cap, cfg.interval, cores)
    value = P / secs
    threads = cores
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": K, "warmup": args.warmup, "ms_per_step": secs * 1e3 / P, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name + ": " + cfg.desc, "minibatch_seqs": cfg.n,
                       "stages": cfg.stages, "t_max_candidates": cfg.K,
                       "t_max_interval": cfg.interval, "per_mb_mem_cap": cfg.mem_cap},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": f"{P} x {cfg.n}-seq mini-batches on {threads} std::threads "
                                       f"(run_plan pool), wall {secs:.1f} s"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "status_ok": int((st == 0).sum())}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--per-gpu", type=int, default=0, help="mini-batches per GPU per step")
    ap.add_argument("--cpu-plans", type=int, default=0, help="cpu_baseline sample size (0: cores)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--streams", type=int, default=3, help="concurrent sub-batches per GPU")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    from paper_2311_10418_b200 import capi, shard
    from paper_2311_10418_b200 import workloads as W

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = W.CONFIGS[args.config]
    M = args.per_gpu or {"C3": 888, "C4": 1536, "C1": 1024, "C2": 192, "C5": 1}.get(cfg.name, 8)
    steps, warm = args.steps, args.warmup
    n = cfg.n
    # distinct mini-batches for every (rank, step): rank r owns groups
    # [r*(W+K), (r+1)*(W+K)) of M consecutive mini-batches of one dataset
    groups = warm + steps
    # rank r draws its own dataset (seed 7 + 1000 r; rank 0's first
    # mini-batch is exactly BASELINE config C3's), so no rank materialises
    # the whole job's samples
    mine = capi.synthetic_dataset(groups * M * n, cfg.max_seq_len, W.SEED + 1000 * rank, W.INPUT_DIST,
                                  W.T5_TARGET_DIST if cfg.encdec else None)
    d_samples = torch.from_numpy(mine).cuda()
    seg = W.seg_offsets(cfg, M)
    d_seg = torch.from_numpy(seg).cuda()
    grid, model = W.grid(), W.model(cfg)
    planner = capi.Planner(local)
    # concurrent sub-batches (pp_tuning::streams): one sub-batch's
    # latency-bound DP overlaps another's cost passes
    planner.set_tuning(streams=args.streams)
    stream = torch.cuda.Stream()
    planner.set_stream(stream.cuda_stream)
    tot = M * n
    dev = torch.device("cuda", local)
    out = {"ordered": torch.empty((tot, 3), dtype=torch.int64, device=dev),
           "splits": torch.empty(tot, dtype=torch.int32, device=dev),
           "mb_times": torch.empty(tot, dtype=torch.float64, device=dev),
           "count": torch.empty(M, dtype=torch.int32, device=dev),
           "t_max_used": torch.empty(M, dtype=torch.float64, device=dev),
           "objective": torch.empty(M, dtype=torch.float64, device=dev),
           "status": torch.empty(M, dtype=torch.int32, device=dev),
           "err_sample_id": torch.empty(M, dtype=torch.int64, device=dev)}
    gather_out = None

    def step(g):
        nonlocal gather_out
        base = g * M * n
        with torch.cuda.stream(stream):
            slot = shard.plan_shard_device(planner, d_samples[base:base + tot], n, M, grid, model,
                                           cfg.stages, 1, cfg.mem_cap, cfg.interval, out, d_seg, seg)
            if world > 1:  # the only collective: one all_gather of the plans per step
                gather_out = shard.gather_plans(slot)

    stats = []
    for g in range(warm):
        step(g)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for g in range(warm, warm + steps):
            step(g)
            stats.append(planner.stats())
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * M * steps / (ms_max / 1e3)
    status_ok = int((out["status"] == 0).sum().item())

    # ---- e2e: host buffers through pp_plan_grid (pinned in, plans out)
    pin = torch.from_numpy(mine).pin_memory()
    pin_np = pin.numpy()
    pinned = []

    def pinned_alloc(shape, dtype):
        t = torch.empty(shape, dtype={np.int64: torch.int64, np.int32: torch.int32,
                                      np.float64: torch.float64}[dtype]).pin_memory()
        pinned.append(t)
        return t.numpy()

    # the plan read back: the ordering as per-segment sample indices (4 B per
    # sample; pp_plan_out.order), splits, micro-batch times and the per-plan scalars
    host_out = capi.Planner.plan_buffers(tot, M, pinned_alloc, order_only=True)
    h2d = tot * 24 + seg.nbytes
    d2h = tot * (4 + 4 + 8) + M * (4 + 8 + 8 + 4 + 8)
    for g in range(warm):
        planner.plan_batch(pin_np[g * tot:(g + 1) * tot], seg, grid, model, cfg.stages, 1, cfg.mem_cap,
                           cfg.interval, out=host_out)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for g in range(warm, warm + steps):
        planner.plan_batch(pin_np[g * tot:(g + 1) * tot], seg, grid, model, cfg.stages, 1, cfg.mem_cap,
                           cfg.interval, out=host_out)
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = world * M * steps / float(te.item())

    # ---- isolated kernel durations: the timed region runs `streams` concurrent
    # sub-batches, so a kernel's event-timed duration there includes the SMs it
    # shares with the other streams' kernels.  A few untimed 1-stream steps give
    # each kernel's duration alone on the GPU (the roofline's isolated figures).
    solo_stats = []
    if args.streams > 1:
        planner.set_tuning(streams=1)
        for g in range(warm, warm + min(steps, 4)):
            step(g)
            solo_stats.append(planner.stats())
        torch.cuda.synchronize()
        planner.set_tuning(streams=args.streams)

    if rank == 0:
        pk, pk_kind = peaks()
        fp64_peak = capi.calibrate_fp64(local) / 1e12  # adds/s -> T ops/s
        def aggregate(sts):
            kern = np.zeros(8)
            launches = np.zeros(8, np.int64)
            agg = {k: 0 for k in ("tr", "ref_tr", "evals", "gen", "sl_a", "sl_b", "bound_tr", "band_b")}
            for s in sts:
                kern += np.array(s["ms_kernel"])
                launches += np.array(s["launches"], np.int64)
                agg["tr"] += s["transitions_executed"]
                agg["ref_tr"] += s["transitions_reference"]
                agg["evals"] += s["candidates_evaluated"]
                agg["gen"] += s["candidates_generated"]
                agg["sl_a"] += s["slices_pass_a"]
                agg["sl_b"] += s["slices_pass_b"]
                agg["bound_tr"] += s["bound_transitions"]
                agg["band_b"] += s["band_bytes"]
            return kern, launches, agg

        kern, launches, agg = aggregate(stats)
        names = capi.KERNEL_NAMES
        kl = W.kind_layouts(cfg)  # (layout, kind) pairs priced per slice
        # algorithmic work per launch category:
        #   pass A: act_mem per (layout, kind): 3 bilinear blends (differences precomputed):
        #           7 FP64 ops + scale = 8 ... counted as 11 with the clamp/compare
        #   pass B: slice time per (layout, kind): 2 blends x 7 + 2 DMUL + 1 DADD = 17 FP64 ops
        #   DP: one 8-byte band entry streamed per transition
        # pass B on sorted single-input (GPT) mini-batches prices each distinct
        # (micro-batch size, padded length) pair once and streams the band out:
        # bound by the band bytes it writes; otherwise by FP64 pricing per slice
        reuse = not cfg.encdec

        def work_of(agg):
            return {
                2: ("fp64", agg["sl_a"] * 11 * kl, "11 FP64 ops per act_mem pricing per (layout, kind)"),
                3: (("hbm", agg["band_b"], "8 B per band entry written (32-row tiles incl. masked entries)")
                    if reuse else ("fp64", agg["sl_b"] * 17 * kl, f"{17 * kl} FP64 ops per band slice")),
                4: ("hbm", agg["bound_tr"] * 8, "8 B band entry per transition"),
                5: ("hbm", (agg["tr"] - agg["bound_tr"]) * 8, "8 B band entry per transition"),
            }

        work = work_of(agg)

        def roof_of(cat, work=work, kern=kern, launches=launches):
            bound, units, algo = work[cat]
            secs = kern[cat] / 1e3
            if bound == "fp64":
                ach, peak, unit = units / secs / 1e12, fp64_peak, "TFLOP/s"
                src = "fp64 add rate measured in-run (pp_calibrate_fp64)"
            else:
                ach, peak, unit = units / secs / 1e9, pk["hbm_gbs"], "GB/s"
                src = f"MEASURED_PEAKS.json hbm_gbs ({pk_kind}, burst)"
            return {"bound": bound, "kernel": names[cat], "achieved": ach, "peak": peak, "unit": unit,
                    "frac": ach / peak, "traffic": None, "algorithmic": algo, "peak_source": src,
                    "avg_launch_ms": kern[cat] / max(int(launches[cat]), 1),
                    "share_of_step": kern[cat] / max(kern.sum(), 1e-9)}

        dom = max(work, key=lambda c: kern[c])
        roof = roof_of(dom)
        # DRAM traffic of the dominant kernel from the committed ncu --set full
        # capture (profiles/<round>/traffic_<config>.json), per launch
        tr = traffic_record(cfg.name)
        if tr and names[dom] in tr["kernels"]:
            per_plan = tr["kernels"][names[dom]]["dram_bytes_per_plan"]
            plans_per_launch = M / max(args.streams, 1)
            roof["traffic"] = per_plan * plans_per_launch
            roof["traffic_source"] = tr["source"]
            if work[dom][0] == "hbm":
                roof["traffic_vs_algorithmic"] = per_plan * M * steps / max(work[dom][1], 1)
        roof["all"] = {names[c]: {k: roof_of(c)[k] for k in ("bound", "achieved", "unit", "frac",
                                                             "share_of_step")}
                       for c in work if kern[c] > 0}
        if solo_stats:
            s_kern, s_launch, s_agg = aggregate(solo_stats)
            s_work = work_of(s_agg)
            iso = {names[c]: {k: roof_of(c, s_work, s_kern, s_launch)[k]
                              for k in ("achieved", "frac", "avg_launch_ms", "share_of_step")}
                   for c in s_work if s_kern[c] > 0}
            roof["isolated"] = {
                "note": (f"the timed region runs {args.streams} concurrent sub-batches, so each kernel's "
                         "event-timed duration includes SMs shared with the other streams; these are the "
                         f"same kernels timed alone ({len(solo_stats)} untimed 1-stream steps, "
                         f"{M} mini-batches each)"),
                "kernels": iso}
            if names[dom] in iso:
                roof["frac_isolated"] = iso[names[dom]]["frac"]
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cores = os.cpu_count() or 1
            cpu = cpu_baseline_sample(cfg, cores, args.cpu_plans or cores)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": warm, "ms_per_step": ms_max / steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name + ": " + cfg.desc, "minibatches_per_gpu_per_step": M,
                       "minibatch_seqs": n, "stages": cfg.stages, "t_max_candidates": cfg.K,
                       "t_max_interval": cfg.interval, "per_mb_mem_cap": cfg.mem_cap,
                       "parallelism": f"mini-batch sharding x{world}, NCCL plan gather",
                       "l2": "distinct mini-batches every step; per-step band traffic > L2 (126 MB)"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": int(launches.sum()),
            "roofline": roof,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "work": {"dp_transitions_per_s": agg["tr"] / (ms_max / 1e3),
                     "reference_equivalent_transitions_per_s": agg["ref_tr"] / (ms_max / 1e3),
                     "candidates_generated": agg["gen"], "dp_passes": agg["evals"],
                     "slices_priced_pass_a": agg["sl_a"], "slices_priced_pass_b": agg["sl_b"],
                     "fp64_add_peak_tops": fp64_peak,
                     "kernel_ms": {nm: float(v) for nm, v in zip(names, kern)},
                     "kernel_launches": {nm: int(v) for nm, v in zip(names, launches)}},
            "status_ok": status_ok,
        }
        print(json.dumps(line), flush=True)
    planner.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
