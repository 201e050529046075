"""Benchmark: micro-batch plans/sec (BASELINE.json metric) at N GPUs of one node.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C1..C5] [--epoch]
    torchrun --nproc-per-node N bench.py --gpus N ...

Default workload: BASELINE config C3 (8192-seq GPT mini-batches, 16 stages,
binding activation-memory cap, 128-candidate t_max sweep).  A "step" plans M
independent mini-batches (order_samples(Sort) + make_slice_cost +
dp_partition each) per GPU with the inputs already resident in HBM and
distinct mini-batches every step (weak scaling), then ONE all_gather of the
packed plans when N > 1.  `--config C4 --epoch` is BASELINE config C4 as
strong scaling: a fixed epoch of 4096 x 2048-seq mini-batches split across
the N GPUs (shard_range), every rank ending with the whole epoch's plans
(splits + per-sample order) after one all_gather.

`--gpus N` without a torchrun environment re-launches itself under
torch.distributed.run with N ranks; under torchrun WORLD_SIZE must equal N.

`e2e` repeats the measurement through the public host-buffer API (pinned
samples in, plans out, copies inside the timed region).  `--impl reference`
times the UNMODIFIED reference planner (oracle/_ref, built from
/root/reference) on the host cores with run_plan's one-mini-batch-per-thread
pool, its inputs built by the reference's own generator / grid / model code.
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
L2_NOTE = "inputs larger than L2: distinct mini-batches every step (no L2 flush)"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """SM clock + throttle-reason sampling DURING the timed region
    (B200_PROFILING.md clocks line).  NVML polled every 2 ms from a thread:
    the timed region is ~0.1-0.2 s, shorter than nvidia-smi's start-up."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index: int):
        self.index = index
        self.sm, self.mask, self.max_mhz = [], 0, None
        self.h = None
        self.stop = threading.Event()

    def _handle(self, nv):
        try:  # the CUDA ordinal's PCI id (NVML ordinals ignore CUDA_VISIBLE_DEVICES)
            import torch
            p = torch.cuda.get_device_properties(self.index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            return nv.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.index)

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = self._handle(nv)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
            self.sample()  # one sample before the region starts: the poller is live
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.h = None
        return self

    def sample(self):
        nv = self.nv
        self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
        self.mask |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))

    def _run(self):
        while not self.stop.wait(0.002):
            try:
                self.sample()
            except Exception:
                return

    def __exit__(self, *a):
        if self.h is not None:
            self.stop.set()
            self.t.join(timeout=2)
            try:
                self.sample()  # and one at the end of the region
            except Exception:
                pass

    def summary(self):
        reasons = sorted(name for name, attr in self.REASONS
                         if self.h is not None and self.mask & int(getattr(self.nv, attr, 0)))
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.sm), "source": "NVML, 2 ms polling over the timed region"}


def traffic_record(config_name):
    """Latest profiles/r*/traffic_<config>.json (per-plan DRAM bytes per kernel
    from an ncu --set full capture), or None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", f"traffic_{config_name.lower()}.json")))
    if not files:
        return None
    with open(files[-1]) as f:
        return json.load(f)


def config_of(cfg, epoch: bool) -> dict:
    """The workload description, IDENTICAL in both arms' lines."""
    c = {"workload": cfg.name + ": " + cfg.desc, "minibatch_seqs": cfg.n, "stages": cfg.stages,
         "t_max_candidates": cfg.K, "t_max_interval": cfg.interval, "per_mb_mem_cap": cfg.mem_cap,
         "l2": L2_NOTE}
    if epoch:
        c["epoch_minibatches"] = cfg.minibatches
    return c


def ref_inputs(ref, cfg, n_minibatches, seed):
    """Inputs built by the REFERENCE's own code (load_dataset,
    ProfileGrid::synthetic, ModelConfig::uniform) — no repo library."""
    from paper_2311_10418_b200.configs import INPUT_DIST, T5_TARGET_DIST

    s = ref.load_dataset(cfg.n * n_minibatches, cfg.max_seq_len, seed, INPUT_DIST,
                         T5_TARGET_DIST if cfg.encdec else None)
    off = np.arange(n_minibatches + 1, dtype=np.int64) * cfg.n
    return s, off, ref.default_grid(), ref.model_uniform(cfg.stages, 2, cfg.encdec)


# --------------------------------------------------------------------- reference
def run_reference(args, rank, world):
    """--impl reference: rank 0 times the reference CPU planner on all host
    cores; the other ranks exit 0 without work."""
    if rank != 0:
        return 0
    from oracle.bind import Reference, reference_available
    from paper_2311_10418_b200.configs import CONFIGS, SEED

    cfg = CONFIGS[args.config]
    if not reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return 0
    cores = os.cpu_count() or 1
    ref = Reference()
    # warm-up: bounded C1 plans through the same code path (page-in)
    c1 = CONFIGS["C1"]
    s1, o1, g1, m1 = ref_inputs(ref, c1, max(args.warmup, 1), SEED)
    ref.plan_batch_timed(s1, o1, g1, m1, c1.stages, 1, c1.mem_cap, c1.interval, min(cores, len(o1) - 1))
    # timed: P = k x cores mini-batches (whole waves of run_plan's pool, one
    # mini-batch per std::thread), k = max(1, K // cores), raised for small
    # configs until the sample is ~10 s of work
    k = max(1, args.steps // cores)
    while True:
        P = cores * k
        s, off, g, m = ref_inputs(ref, cfg, P, SEED)
        secs, tm, ob, cnt, st = ref.plan_batch_timed(s, off, g, m, cfg.stages, 1, cfg.mem_cap, cfg.interval,
                                                     cores)
        if secs >= 5.0 or k >= 256:
            break
        k = min(256, k * max(2, math.ceil(10.0 / max(secs, 1e-3))))
    value = P / secs
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs * 1e3 / P,
            "higher_is_better": True, "scaling": "strong" if args.epoch else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": config_of(cfg, args.epoch),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                             "sample": f"{P} x {cfg.n}-seq mini-batches of {cfg.name} on {cores} std::threads "
                                       f"(run_plan pool, {P // cores} wave(s)), wall {secs:.1f} s"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "status_ok": int((st == 0).sum())}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------ cpu baseline leg
def cpu_baseline_and_parity(planner, cfg, samples, plans, cores, grid, model):
    """The unmodified reference (oracle/_ref) plans the FIRST `plans`
    mini-batches of the benchmark's own workload on all host cores
    (run_plan's pool); the device planner plans the same mini-batches through
    the public host API and every plan is compared bit for bit."""
    from oracle.bind import Reference, reference_available

    if not reference_available():
        return None, None
    ref = Reference()
    s = samples[:plans * cfg.n]
    off = np.arange(plans + 1, dtype=np.int64) * cfg.n
    r = ref.plan_batch_full(s, off, grid, model, cfg.stages, 1, cfg.mem_cap, cfg.interval, cores)
    secs = r["seconds"]
    cpu = {"value": plans / secs, "unit": UNIT, "cores": cores, "kind": "reference",
           "sample": f"{plans} x {cfg.n}-seq mini-batches of {cfg.name} (the first of this run's workload), "
                     f"one per std::thread (run_plan pool), wall {secs:.1f} s"}
    d = planner.plan_batch(s, off, grid, model, cfg.stages, 1, cfg.mem_cap, cfg.interval)
    bad = []
    for k in range(plans):
        m = int(d["count"][k])
        sl = slice(off[k], off[k] + m)
        same = (int(d["status"][k]) == int(r["status"][k]) and m == int(r["count"][k])
                and d["t_max_used"][k] == r["t_max_used"][k] and d["objective"][k] == r["objective"][k]
                and np.array_equal(d["splits"][sl], r["splits"][sl])
                and d["mb_times"][sl].tobytes() == r["mb_times"][sl].tobytes()
                and np.array_equal(d["ordered"][off[k]:off[k + 1], 0], r["ordered_ids"][off[k]:off[k + 1]]))
        if not same:
            bad.append(k)
    parity = {"checked": plans, "mismatches": len(bad), "first_mismatch": bad[0] if bad else None,
              "against": "oracle/_ref (unmodified reference) on the same mini-batches",
              "fields": "status, count, splits, mb_times (bits), t_max_used (bits), objective (bits), ordered ids"}
    return cpu, parity


# --------------------------------------------------------------------- ours
def run_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist

    from paper_2311_10418_b200 import capi, shard
    from paper_2311_10418_b200 import workloads as W

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # NCCL's init log on stderr shows the rank count of the communicator
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=dev)
    cfg = W.CONFIGS[args.config]
    epoch = args.epoch
    n = cfg.n
    steps, warm = args.steps, args.warmup
    grid, model = W.grid(), W.model(cfg)
    if epoch:
        # strong scaling: the fixed epoch, rank r plans shard_range(...) of it
        M_total = cfg.minibatches
        lo, hi = shard.shard_range(M_total, world, rank)
        M = hi - lo
        # distinct epochs rotated across steps so a step's inputs were not
        # touched by the previous step (seed 7 + e; e = 0 is BASELINE's C4)
        shard_bytes = M * n * 24
        E = max(2, math.ceil(2 * 126e6 / max(shard_bytes, 1)) + 1)
        E = min(E, warm + steps)
        parts = []
        for e in range(E):
            full = capi.synthetic_dataset(M_total * n, cfg.max_seq_len, W.SEED + e, W.INPUT_DIST,
                                          W.T5_TARGET_DIST if cfg.encdec else None)
            parts.append(full[lo * n:hi * n].copy())
        mine = np.concatenate(parts)
        groups = E
    else:
        M = args.per_gpu or {"C3": 888, "C4": 1536, "C1": 1024, "C2": 192, "C5": 1}.get(cfg.name, 8)
        M_total = M * world
        groups = warm + steps
        # rank r draws its own dataset (seed 7 + 1000 r; rank 0's first
        # mini-batch is exactly BASELINE config C3's)
        mine = capi.synthetic_dataset(groups * M * n, cfg.max_seq_len, W.SEED + 1000 * rank, W.INPUT_DIST,
                                      W.T5_TARGET_DIST if cfg.encdec else None)
    d_samples = torch.from_numpy(mine).to(dev)
    seg = np.arange(M + 1, dtype=np.int64) * n
    planner = capi.Planner(local)
    planner.set_tuning(streams=args.streams)
    stream = torch.cuda.Stream(device=dev)
    planner.set_stream(stream.cuda_stream)
    tot = M * n
    out = {"ordered": torch.empty((tot, 3), dtype=torch.int64, device=dev),
           "order": torch.empty(tot, dtype=torch.int32, device=dev),
           "splits": torch.empty(tot, dtype=torch.int32, device=dev),
           "mb_times": torch.empty(tot, dtype=torch.float64, device=dev),
           "count": torch.empty(M, dtype=torch.int32, device=dev),
           "t_max_used": torch.empty(M, dtype=torch.float64, device=dev),
           "objective": torch.empty(M, dtype=torch.float64, device=dev),
           "status": torch.empty(M, dtype=torch.int32, device=dev),
           "err_sample_id": torch.empty(M, dtype=torch.int64, device=dev)}
    words = shard.slot_words(n, True)
    slots = torch.empty((M, words), dtype=torch.int64, device=dev)
    gathered = {}
    # planning calls of at most `chunk` mini-batches (bounded scratch per call)
    chunk = min(M, args.chunk) if args.chunk > 0 else M
    seg_c = np.arange(chunk + 1, dtype=np.int64) * n
    d_seg_c = torch.from_numpy(seg_c).to(dev)
    per_sample = ("ordered", "order", "splits", "mb_times")

    # concurrent callers (one GPU, no collective): caller c has its own
    # context, stream and output buffers and plans steps c, c + C, ... from
    # its own host thread — run_plan's pool pattern; caller 0 is `planner`
    # (one caller for very long mini-batches: each pass is already a
    # whole-GPU cooperative kernel, and a context holds a multi-GB band)
    callers = max(1, args.callers) if (world == 1 and not epoch and cfg.n < 16384) else 1
    args.callers_used = callers
    cplans, cstreams, couts, cslots = [planner], [stream], [out], [slots]
    for _ in range(callers - 1):
        pl = capi.Planner(local)
        st_c = torch.cuda.Stream(device=dev)
        pl.set_stream(st_c.cuda_stream)
        cplans.append(pl)
        cstreams.append(st_c)
        couts.append({k: torch.empty_like(v) for k, v in out.items()})
        cslots.append(torch.empty_like(slots))
    for pl in cplans:
        pl.set_tuning(streams=args.caller_streams if callers > 1 else args.streams)

    def plan_into(src, c=0):
        pl, o_all, sl_all = cplans[c], couts[c], cslots[c]
        for c0 in range(0, M, chunk):
            mc = min(chunk, M - c0)
            o = {k: (v[c0 * n:(c0 + mc) * n] if k in per_sample else v[c0:c0 + mc]) for k, v in o_all.items()}
            shard.plan_shard_device(pl, src[c0 * n:(c0 + mc) * n], n, mc, grid, model, cfg.stages, 1,
                                    cfg.mem_cap, cfg.interval, o, d_seg_c[:mc + 1], seg_c[:mc + 1],
                                    sl_all[c0:c0 + mc])
        return sl_all

    def step(g, c=0):
        base = (g % groups) * tot
        with torch.cuda.stream(cstreams[c]):
            sl = plan_into(d_samples[base:base + tot], c)
            if world > 1:  # the only collective: one all_gather of the plans per step
                gathered["slots"] = (shard.gather_epoch(sl, M_total) if epoch else shard.gather_plans(sl))

    for g in range(warm):
        step(g)
    for c in range(1, callers):
        step(c, c)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    stats = []
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        if callers == 1:
            for g in range(warm, warm + steps):
                step(g)
                stats.append(planner.stats())
        else:
            per = [[] for _ in range(callers)]
            errs = []

            def run(c):
                try:
                    cstreams[c].wait_event(ev0)
                    for g in range(warm + c, warm + steps, callers):
                        step(g, c)
                        per[c].append(cplans[c].stats())
                except BaseException as e:  # noqa: BLE001 - re-raised below
                    errs.append(e)

            ths = [threading.Thread(target=run, args=(c,)) for c in range(callers)]
            for th in ths:
                th.start()
            for th in ths:
                th.join()
            if errs:
                raise errs[0]
            for c in range(1, callers):
                stream.wait_stream(cstreams[c])
            stats = [x for p_ in per for x in p_]
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    units_per_step = M_total  # every rank's mini-batches (epoch: the whole epoch)
    value = units_per_step * steps / (ms_max / 1e3)
    status_ok = int((out["status"] == 0).sum().item())
    if world > 1:
        g_st = gathered["slots"][:, 1]
        gathered_ok = int((g_st == 0).sum().item())
    else:
        gathered_ok = status_ok

    # ---- e2e through the public API with host buffers
    if epoch or world > 1:
        # pinned shard in -> plan -> pack -> all_gather -> the gathered plans
        # out, all on the stream inside the timed region
        pin = torch.from_numpy(mine[:tot]).pin_memory()
        h_out = torch.empty((M_total if world > 1 else M, words), dtype=torch.int64).pin_memory()
        d_in = torch.empty((tot, 3), dtype=torch.int64, device=dev)

        def e2e_step():
            with torch.cuda.stream(stream):
                d_in.copy_(pin, non_blocking=True)
                sl = plan_into(d_in)
                res = (shard.gather_epoch(sl, M_total) if epoch else shard.gather_plans(sl)) if world > 1 else sl
                h_out.copy_(res, non_blocking=True)

        for _ in range(warm):
            e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_value = units_per_step * steps / (float(te.item()) / 1e3)
        h2d, d2h = tot * 24, h_out.numel() * 8
        e2e_api = "pinned shard -> Planner.plan_batch_device + pp_pack_plan_slots (+ all_gather) -> pinned plans"
    else:
        # pp_plan_grid: pinned samples in, plans (order indices, splits, times,
        # scalars) out; the library pipelines its own copies
        pin = torch.from_numpy(mine).pin_memory()
        pin_np = pin.numpy()
        pinned = []

        def pinned_alloc(shape, dtype):
            tt = torch.empty(shape, dtype={np.int64: torch.int64, np.int32: torch.int32,
                                           np.float64: torch.float64}[dtype]).pin_memory()
            pinned.append(tt)
            return tt.numpy()

        host_out = capi.Planner.plan_buffers(tot, M, pinned_alloc, order_only=True)
        h2d = tot * 24 + seg.nbytes
        d2h = tot * (4 + 4 + 8) + M * (4 + 8 + 8 + 4 + 8)
        # one caller: the library's own host pipeline (--streams workers);
        # several callers: --e2e-streams each (default 1: the callers are the pipeline)
        e2e_streams = args.e2e_streams or 1
        planner.set_tuning(streams=args.streams)
        for g in range(warm):
            planner.plan_batch(pin_np[g * tot:(g + 1) * tot], seg, grid, model, cfg.stages, 1, cfg.mem_cap,
                               cfg.interval, out=host_out)
        t0 = time.perf_counter()
        for g in range(warm, warm + steps):
            planner.plan_batch(pin_np[g * tot:(g + 1) * tot], seg, grid, model, cfg.stages, 1, cfg.mem_cap,
                               cfg.interval, out=host_out)
        e2e_single = M * steps / (time.perf_counter() - t0)
        e2e_value = e2e_single
        e2e_api = "pp_plan_grid (host buffers; pinned samples in, plans out)"
        callers = max(1, args.e2e_callers) if cfg.n < 16384 else 1
        if callers > 1:
            # concurrent callers, as the reference's run_plan drives
            # plan_iteration from a thread pool: caller c plans steps
            # c, c + C, ... through its own context and pinned buffers, so one
            # call's uploads and downloads overlap another's planning
            plans = [planner] + [capi.Planner(local) for _ in range(callers - 1)]
            for pl in plans:
                pl.set_tuning(streams=e2e_streams)
            outs = [host_out] + [capi.Planner.plan_buffers(tot, M, pinned_alloc, order_only=True)
                                 for _ in range(callers - 1)]
            for c in range(callers):  # (warm-up of every context at this tuning)
                plans[c].plan_batch(pin_np[:tot], seg, grid, model, cfg.stages, 1, cfg.mem_cap, cfg.interval,
                                    out=outs[c])
            errs = []

            def caller(c):
                try:
                    for g in range(warm + c, warm + steps, callers):
                        plans[c].plan_batch(pin_np[g * tot:(g + 1) * tot], seg, grid, model, cfg.stages, 1,
                                            cfg.mem_cap, cfg.interval, out=outs[c])
                except BaseException as e:  # noqa: BLE001 - re-raised below
                    errs.append(e)

            ths = [threading.Thread(target=caller, args=(c,)) for c in range(callers)]
            t0 = time.perf_counter()
            for th in ths:
                th.start()
            for th in ths:
                th.join()
            e2e_value = M * steps / (time.perf_counter() - t0)
            if errs:
                raise errs[0]
            for pl in plans[1:]:
                pl.close()
            e2e_api = {"api": f"pp_plan_grid (host buffers; pinned samples in, plans out) from {callers} "
                              f"concurrent host threads (one context each, streams={e2e_streams}), step g on "
                              "thread g mod callers: run_plan's pool pattern",
                       "callers": callers, "single_caller_value": e2e_single,
                       "single_caller_streams": args.streams}
        # pinned outputs: splits / mb_times come back as each segment's valid
        # prefix (count[s] entries, prefix_out_kernel), the order in full
        d2h = tot * 4 + int(host_out["count"].astype(np.int64).sum()) * (4 + 8) + M * (4 + 8 + 8 + 4 + 8)

    # ---- isolated kernel durations: the timed region runs `streams` concurrent
    # sub-batches, so per-kernel event spans there overlap and are NOT
    # durations; a few untimed 1-stream steps give each kernel's average launch
    # duration alone on the GPU (the roofline's numbers).
    solo_stats = []
    planner.set_tuning(streams=1)
    for g in range(warm, warm + min(steps, 4)):
        step(g)
        solo_stats.append(planner.stats())
    torch.cuda.synchronize()
    planner.set_tuning(streams=args.streams)

    line = None
    if rank == 0:
        line = report(args, cfg, W, capi, planner, stats, solo_stats, M, M_total, world, steps, warm, ms_max,
                      value, clk, e2e_value, e2e_api, h2d, d2h, status_ok, gathered_ok, mine, local)
        print(json.dumps(line), flush=True)
    planner.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def report(args, cfg, W, capi, planner, stats, solo_stats, M, M_total, world, steps, warm, ms_max, value, clk,
           e2e_value, e2e_api, h2d, d2h, status_ok, gathered_ok, mine, local):
    import torch

    pk, pk_kind = peaks()
    names = capi.KERNEL_NAMES

    def aggregate(sts):
        kern = np.zeros(8)
        launches = np.zeros(8, np.int64)
        agg = {k: 0 for k in ("tr", "ref_tr", "evals", "gen", "ref_ev", "sl_a", "sl_b", "bound_tr", "band_b")}
        for s in sts:
            kern += np.array(s["ms_kernel"])
            launches += np.array(s["launches"], np.int64)
            agg["tr"] += s["transitions_executed"]
            agg["ref_tr"] += s["transitions_reference"]
            agg["evals"] += s["candidates_evaluated"]
            agg["gen"] += s["candidates_generated"]
            agg["ref_ev"] += s["candidates_ref_evaluated"]
            agg["sl_a"] += s["slices_pass_a"]
            agg["sl_b"] += s["slices_pass_b"]
            agg["bound_tr"] += s["bound_transitions"]
            agg["band_b"] += s["band_bytes"]
        return kern, launches, agg

    kern, launches, agg = aggregate(stats)
    s_kern, s_launch, s_agg = aggregate(solo_stats)
    fp64_peak = capi.calibrate_fp64(local) / 1e12  # adds/s -> T ops/s
    kl = W.kind_layouts(cfg)
    reuse = not cfg.encdec

    # algorithmic work per kernel category
    table = s_agg["band_b"] == 0 and reuse  # the call's slice table (gtab.cu): no band in HBM
    samples = len(solo_stats) * M * cfg.n
    props = torch.cuda.get_device_properties(local)
    clk_sum = clk.summary()
    sm_mhz = clk_sum["sm_mhz"] or clk_sum["sm_max_mhz"] or pk.get("sm_max_mhz", 1965.0)

    def work_of(a):
        w = {
            0: ("hbm", samples * 68, "68 B per sample: 24 B record in, 24 B ordered record + 16 B SoA lengths "
                                     "+ 4 B order out (sort.cu)"),
            2: ("fp64", a["sl_a"] * 11 * kl, "11 FP64 ops per act_mem pricing per (layout, kind)"),
            3: (("hbm", a["band_b"], "8 B per band entry written (32-row tiles incl. masked entries)")
                if reuse else ("fp64", a["sl_b"] * 17 * kl, f"{17 * kl} FP64 ops per band slice")),
        }
        if table:
            # DP transitions read the L2-resident slice table: the bound is the
            # SM issue rate; SURVEY §8(d) prices a transition at ~7 thread
            # instructions (one add + compares + select)
            w[4] = ("issue", a["bound_tr"] * 7 / 32, "7 thread-instructions per DP transition (SURVEY §8d)")
            w[5] = ("issue", (a["tr"] - a["bound_tr"]) * 7 / 32, "7 thread-instructions per DP transition")
        else:
            w[4] = ("hbm", a["bound_tr"] * 8, "8 B band entry per transition")
            w[5] = ("hbm", (a["tr"] - a["bound_tr"]) * 8, "8 B band entry per transition")
        return w

    work = work_of(s_agg)

    def roof_of(cat):
        bound, units, algo = work[cat]
        secs = s_kern[cat] / 1e3
        if bound == "fp64":
            ach, peak, unit = units / secs / 1e12, fp64_peak, "TFLOP/s"
            src = "fp64 add rate measured in-run (pp_calibrate_fp64)"
        elif bound == "issue":
            ach, unit = units / secs / 1e9, "G warp-instr/s"
            peak = 4 * props.multi_processor_count * sm_mhz / 1e3
            src = (f"4 warp-instructions per cycle per SM x {props.multi_processor_count} SMs x "
                   f"{sm_mhz:.0f} MHz (SM clock measured over the timed region)")
        else:
            ach, peak, unit = units / secs / 1e9, pk["hbm_gbs"], "GB/s"
            src = f"MEASURED_PEAKS.json hbm_gbs ({pk_kind}, burst)"
        return {"bound": bound, "kernel": names[cat], "achieved": ach, "peak": peak, "unit": unit,
                "frac": ach / peak, "traffic": None, "algorithmic": algo, "peak_source": src,
                "avg_launch_ms": s_kern[cat] / max(int(s_launch[cat]), 1),
                "share_of_step": s_kern[cat] / max(s_kern.sum(), 1e-9)}

    # (slice table: category 3 is the table build + candidate scan, no band bytes to price)
    cats = [c for c in work if s_kern[c] > 0 and not (table and c == 3)]
    dom = max((c for c in cats if c != 0), key=lambda c: s_kern[c])
    roof = roof_of(dom)
    roof["timing"] = (f"per-launch durations from {len(solo_stats)} untimed one-stream steps of {M} mini-batches "
                      "(CUDA events on the launching stream, each kernel alone on the GPU)")
    tr = traffic_record(cfg.name)
    if tr and names[dom] in tr["kernels"]:
        rec = tr["kernels"][names[dom]]
        per_plan = rec["dram_bytes_per_plan"]
        roof["traffic"] = per_plan * M
        roof["traffic_source"] = tr["source"]
        if work[dom][0] == "hbm":
            roof["traffic_vs_algorithmic"] = per_plan * M * len(solo_stats) / max(work[dom][1], 1)
        for k in ("ncu_issue_active_pct", "ncu_warp_instr_per_transition", "ncu_ipc", "ncu_l2_hit_pct"):
            if k in rec:
                roof[k] = rec[k]
    if 0 in cats:
        roof["sort"] = {k: roof_of(0)[k] for k in ("bound", "achieved", "peak", "unit", "frac", "algorithmic",
                                                   "avg_launch_ms")}
        if tr and names[0] in tr["kernels"]:
            roof["sort"]["traffic"] = tr["kernels"][names[0]]["dram_bytes_per_plan"] * M
    roof["all"] = {names[c]: {k: roof_of(c)[k] for k in ("bound", "achieved", "unit", "frac", "avg_launch_ms",
                                                         "share_of_step")} for c in cats}
    cpu = parity = None
    if world == 1 and not args.no_cpu_baseline and cfg.name == "C5":
        # the reference's dp_partition at n = 65,536 builds two
        # 34 GB triangular tables and runs ~9 h per plan; parity is pinned by
        # the streaming restatement instead (tests/golden/c5.json)
        cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count() or 1, "kind": "reference",
               "sample": "not runnable: ~9 h and >= 34 GB of tables per 65,536-seq plan (SURVEY.md §8d); "
                         "C5 parity: tests/golden/c5.json from the streaming C restatement"}
    elif world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        solo = capi.Planner(local)
        cpu, parity = cpu_baseline_and_parity(solo, cfg, mine, args.cpu_plans or cores, cores, W.grid(),
                                              W.model(cfg))
        solo.close()
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
        "warmup": warm, "ms_per_step": ms_max / steps, "higher_is_better": True,
        "scaling": "strong" if args.epoch else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(cfg, args.epoch),
        "setup": {"minibatches_per_gpu_per_step": M, "minibatches_per_step": M_total,
                  "parallelism": (f"epoch sharded x{world} (shard_range), one NCCL all_gather of plan slots"
                                  if args.epoch else f"mini-batch sharding x{world}, NCCL plan gather"),
                  "concurrent_sub_batches": args.streams,
                  "device_callers": getattr(args, "callers_used", 1),
                  "device_caller_streams": args.caller_streams if getattr(args, "callers_used", 1) > 1
                  else args.streams},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                **(e2e_api if isinstance(e2e_api, dict) else {"api": e2e_api})},
        "gpu_launches": int(launches.sum()) + int(launches[0]),  # + one slot-pack kernel per planning call
        "roofline": roof,
        "cpu_baseline": cpu,
        "parity": parity,
        "clocks": clk.summary(),
        "work": {"dp_transitions_per_s": agg["tr"] / (ms_max / 1e3),
                 "reference_equivalent_transitions_per_s": agg["ref_tr"] / (ms_max / 1e3),
                 "candidates_generated": agg["gen"], "candidates_reference_loop": agg["ref_ev"],
                 "dp_passes": agg["evals"],
                 "slices_priced_pass_a": agg["sl_a"], "slices_priced_pass_b": agg["sl_b"],
                 "fp64_add_peak_tops": fp64_peak,
                 "kernel_event_spans_ms_overlapped": {nm: float(v) for nm, v in zip(names, kern)},
                 "kernel_launches": {nm: int(v) for nm, v in zip(names, launches)}},
        "status_ok": status_ok, "gathered_status_ok": gathered_ok,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--epoch", action="store_true", help="C4 whole-epoch strong scaling")
    ap.add_argument("--per-gpu", type=int, default=0, help="mini-batches per GPU per step (weak mode)")
    ap.add_argument("--cpu-plans", type=int, default=0, help="cpu_baseline / parity sample (0: cores)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--streams", type=int, default=3, help="concurrent sub-batches per planning call")
    ap.add_argument("--callers", type=int, default=8,
                    help="device-resident measurement: host threads issuing planning calls (alternate steps)")
    ap.add_argument("--caller-streams", type=int, default=1, help="streams per call with --callers > 1")
    ap.add_argument("--e2e-streams", type=int, default=1, help="streams of each concurrent e2e caller")
    ap.add_argument("--e2e-callers", type=int, default=8,
                    help="host threads issuing the e2e pp_plan_grid calls (alternate steps)")
    ap.add_argument("--chunk", type=int, default=0, help="mini-batches per planning call (0: all; epoch: 1024)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.epoch and args.config != "C4":
        ap.error("--epoch plans BASELINE config C4's fixed epoch (use --config C4)")
    if args.epoch and args.chunk == 0:
        args.chunk = 1024

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # self-launch: one rank per GPU under torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 1000),
               os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        return 2
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
