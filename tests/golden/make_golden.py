"""Generate the golden parity fixtures from the UNMODIFIED reference planner.

Run in the build container (needs /root/reference to build oracle/_ref):
    python tests/golden/make_golden.py
Writes tests/golden/{toy,grid,c1}.json.  Doubles are stored as float.hex()
strings so the fixtures pin results bit-exactly.

Cases:
  toy  : the hot-path known answers of proj/tests/test_microbatch.cpp
         (:139-178, :246-268) plus seeded random toy instances in the style of
         :180-244 and acceptance.cpp:80-121 (t(M) = max_len*|M|, mem = k*|M|),
         run through the reference's dp_partition with a generic SliceCostFn.
  grid : seeded synthetic mini-batches through order_samples(Sort) ->
         make_slice_cost -> dp_partition over GPT / T5 layouts, stage counts,
         replica counts, binding and non-binding caps, quantized and exact
         candidate sets.
  c1   : BASELINE config 1 (256 sequences, 4 stages, 32 candidates).
"""
from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.bind import Reference, build  # noqa: E402
from paper_2311_10418_b200 import capi  # noqa: E402
from paper_2311_10418_b200 import workloads as W  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def hx(x: float) -> str:
    return float(x).hex()


def toy_tables(lens, mem_per_sample=0.0, heavy=False):
    n = len(lens)
    T, M = [], []
    for i in range(n):
        mx = 0
        for j in range(i + 1, n + 1):
            mx = max(mx, lens[j - 1])
            t = float(mx) * float(j - i)
            T.append(t)
            M.append(t if heavy else mem_per_sample * float(j - i))
    return np.array(T), np.array(M)


def plan_record(p, ordered=None):
    rec = {"status": int(p.status), "err_sample_id": int(p.err_sample_id)}
    if p.status == 0:
        rec.update(splits=[int(x) for x in p.splits], mb_times=[hx(x) for x in p.mb_times],
                   t_max_used=hx(p.t_max_used), objective=hx(p.objective),
                   replica=[int(x) for x in p.replica], max_load=hx(p.max_load))
        if ordered is not None:
            rec["ordered_ids"] = [int(x) for x in ordered[:, 0]]
    return rec


def toy_cases(ref):
    cases = []

    def add(name, lens, c, d=1, cap=math.inf, interval=0.0, mem=0.0, heavy=False):
        T, M = toy_tables(lens, mem, heavy)
        p = ref.plan_tables(T, M, len(lens), c, d, cap, interval)
        cases.append(dict(name=name, lens=list(map(int, lens)), mem_per_sample=mem, heavy=heavy,
                          stage_count=c, replica_count=d, mem_cap=hx(cap), t_max_interval=hx(interval),
                          expect=plan_record(p)))

    # known answers transcribed from proj/tests/test_microbatch.cpp
    add("worked_instance_:139", [1, 1, 2, 8], 2)            # objective 20, splits {2,3,4}
    add("single_sample_:157", [7], 4)                       # objective 28
    add("memory_cap_:168", [4, 4, 4, 4], 1, cap=2.0, mem=1.0)   # objective 16
    add("cap_admits_singletons_:246", [2, 9, 3], 1, cap=5.0, mem=1.0)
    add("infeasible_sample_:262", [2, 9, 3], 1, cap=5.0, heavy=True)  # sample_id 1
    add("replica_load_:292", [1, 1, 2, 8], 2, d=2)          # max_replica_load 8
    rng = np.random.default_rng(123)
    for k in range(120):  # brute-force style (:180-200, acceptance.cpp:80-121)
        n = int(rng.integers(1, 13))
        lens = rng.integers(1, 65, n).tolist()
        for c in (1, 2, 4):
            for d in (1, 2):
                add(f"random_exact_{k}_c{c}_d{d}", lens, c, d)
    for k in range(40):  # caps + quantized candidates (:202-244)
        n = int(rng.integers(2, 15))
        lens = rng.integers(1, 51, n).tolist()
        add(f"random_cap_{k}", lens, 3, cap=4.0, interval=5.0, mem=1.0)
        add(f"random_cap_tight_{k}", lens, 2, cap=2.0, interval=0.0, mem=1.0)
    for k in range(40):  # tie-heavy: few distinct lengths
        n = int(rng.integers(3, 20))
        lens = rng.integers(1, 4, n).tolist()
        add(f"ties_{k}", lens, int(rng.integers(1, 6)), int(rng.integers(1, 3)),
            interval=float(rng.choice([0.0, 1.0, 2.0])))
    return cases


def grid_cases(ref):
    cases = []
    grid = capi.synthetic_grid()
    rng = np.random.default_rng(2024)
    seed = 100
    for n in (1, 2, 3, 5, 17, 40, 64, 130):
        for encdec in (False, True):
            for C in (1, 2, 4, 16):
                seed += 1
                samples = capi.synthetic_dataset(n, 8192, seed, W.INPUT_DIST,
                                                 W.T5_TARGET_DIST if encdec else None)
                # shuffle ids so the sort has work to do
                samples[:, 0] = rng.permutation(n) + 1000
                model = capi.Model.uniform(C, 2, encdec)
                for mode in ("inf5", "exact", "kq", "cap", "d2"):
                    cap, interval, d = math.inf, 5.0, 1
                    if mode == "exact":
                        interval = 0.0
                    if mode in ("kq", "cap", "d2"):
                        o = ref.order_samples(samples)
                        big = ref.plan(o, grid, model, 1, 1, math.inf, 0.0, presorted=True)
                        tot = float(np.sum(big.mb_times)) if big.status == 0 else 1.0
                        interval = max(tot / 16.0, 1e-3)
                    if mode == "cap":
                        acts = [capi.slice_cost_host(grid, model, ref.order_samples(samples), k, k + 1)[1]
                                for k in range(n)]
                        cap = float(rng.choice([1.0, 2.0, 3.5])) * max(acts)
                    if mode == "d2":
                        d = 2
                    p = ref.plan(samples, grid, model, C, d, cap, interval)
                    cases.append(dict(name=f"grid_n{n}_{'t5' if encdec else 'gpt'}_c{C}_{mode}",
                                      n=n, seed=seed, encdec=encdec, stages=C, replica_count=d,
                                      mem_cap=hx(cap), t_max_interval=hx(interval),
                                      samples=samples.tolist(), expect=plan_record(p, p.ordered)))
    # infeasible singleton under a cap below the largest sample
    samples = capi.synthetic_dataset(30, 8192, 5, W.INPUT_DIST, None)
    model = capi.Model.uniform(4, 2, False)
    o = ref.order_samples(samples)
    acts = [capi.slice_cost_host(grid, model, o, k, k + 1)[1] for k in range(30)]
    cap = 0.5 * (sorted(acts)[-1] + sorted(acts)[-2])
    p = ref.plan(samples, grid, model, 4, 1, cap, 5.0)
    cases.append(dict(name="grid_infeasible_sample", n=30, seed=5, encdec=False, stages=4,
                      replica_count=1, mem_cap=hx(cap), t_max_interval=hx(5.0),
                      samples=samples.tolist(), expect=plan_record(p, p.ordered)))
    return cases


def c1_case(ref):
    cfg = W.CONFIGS["C1"]
    samples = W.dataset(cfg, 1)
    p = ref.plan(samples, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
    return dict(name="C1", config="C1", expect=plan_record(p, p.ordered))


def main():
    build(ref=True)
    ref = Reference()
    with open(os.path.join(OUT, "toy.json"), "w") as f:
        json.dump(toy_cases(ref), f, separators=(",", ":"))
    with open(os.path.join(OUT, "grid.json"), "w") as f:
        json.dump(grid_cases(ref), f, separators=(",", ":"))
    with open(os.path.join(OUT, "c1.json"), "w") as f:
        json.dump(c1_case(ref), f, separators=(",", ":"))
    for k in ("toy", "grid", "c1"):
        print(k, os.path.getsize(os.path.join(OUT, k + ".json")), "bytes")




def c3_main():
    """C3 golden (slow: ~2 min of reference CPU time).  python make_golden.py c3"""
    ref = Reference()
    cfg = W.CONFIGS["C3"]
    samples = W.dataset(cfg, 1)
    p = ref.plan(samples, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
    rec = plan_record(p, None)
    rec["ordered_ids"] = [int(x) for x in p.ordered[:, 0]]
    with open(os.path.join(OUT, "c3.json"), "w") as f:
        json.dump(dict(name="C3", config="C3", expect=rec), f, separators=(",", ":"))


def c5_main():
    """C5 golden from the STREAMING restatement (oracle/pp_stream.c; the
    reference itself needs ~9 h and 34 GB of tables at n = 65,536).  The
    restatement is pinned against the unmodified reference at n <= 2048 by
    tests/test_oracle.py::test_stream_restatement_matches_reference.
        python tests/golden/make_golden.py c5        (~2 min on 8 cores)"""
    import hashlib
    import time

    from oracle.bind import Oracle

    cfg = W.CONFIGS["C5"]
    samples = W.dataset(cfg, 1)
    t0 = time.time()
    p = Oracle().plan_stream(samples, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
    secs = time.time() - t0
    assert p.status == 0
    sp = np.asarray(p.splits, np.int64)
    rec = {"status": 0, "count": int(len(sp)),
           "split_deltas": [int(x) for x in np.diff(np.concatenate([[0], sp]))],
           "mb_times_sha256": hashlib.sha256(np.ascontiguousarray(p.mb_times, "<f8").tobytes()).hexdigest(),
           "mb_time_first": [hx(x) for x in p.mb_times[:8]], "mb_time_max": hx(float(np.max(p.mb_times))),
           "t_max_used": hx(p.t_max_used), "objective": hx(p.objective),
           "ordered_ids_sha256": hashlib.sha256(np.ascontiguousarray(p.ordered[:, 0], "<i8").tobytes()).hexdigest(),
           "n_candidates": p.n_candidates, "n_evaluated": p.n_evaluated}
    with open(os.path.join(OUT, "c5.json"), "w") as f:
        json.dump(dict(name="C5", config="C5", generator="oracle/pp_stream.c (orc_plan_grid_stream)",
                       seconds=round(secs, 1), expect=rec), f, separators=(",", ":"))
    print("c5", len(sp), "micro-batches,", p.n_candidates, "candidates,", p.n_evaluated, "evaluated,",
          f"{secs:.0f} s")


if __name__ == "__main__":
    if sys.argv[1:] == ["c3"]:
        c3_main()
    elif sys.argv[1:] == ["c5"]:
        c5_main()
    else:
        main()
