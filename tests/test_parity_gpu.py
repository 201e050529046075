"""GPU parity: the sm_100a planner through the C-ABI against the golden
fixtures (generated from the unmodified reference) and the C restatement.
Bit-exact on splits, per-micro-batch times, ordering and t_max_used;
objective within 1e-6 relative (BASELINE.json north_star), in practice equal."""
import math

import numpy as np
import pytest

from conftest import assert_plan_matches, load_golden, record, toy_tables, unhex
from oracle.bind import Oracle, Reference, reference_available
from paper_2311_10418_b200 import capi
from paper_2311_10418_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def planner():
    p = capi.Planner(0)
    yield p
    p.close()


@pytest.fixture(scope="module")
def orc():
    return Oracle()


def _plan_or_status(fn):
    try:
        return fn()
    except capi.InfeasibleError as e:
        return capi.Plan(capi.PP_ERR_INFEASIBLE_SAMPLE if e.sample_id >= 0 else capi.PP_ERR_INFEASIBLE,
                         err_sample_id=e.sample_id)


def test_golden_toy_tables(planner):
    for case in load_golden("toy"):
        T, M = toy_tables(case["lens"], case["mem_per_sample"], case["heavy"])
        p = _plan_or_status(lambda: planner.plan_tables(
            T, M, len(case["lens"]), case["stage_count"], case["replica_count"],
            unhex(case["mem_cap"]), unhex(case["t_max_interval"])))
        assert_plan_matches(p, case["expect"], case["name"])


def test_golden_grid(planner):
    grid = capi.synthetic_grid()
    for case in load_golden("grid"):
        model = capi.Model.uniform(case["stages"], 2, case["encdec"])
        s = np.array(case["samples"], np.int64)
        p = _plan_or_status(lambda: planner.plan(s, grid, model, case["stages"], case["replica_count"],
                                                 unhex(case["mem_cap"]), unhex(case["t_max_interval"])))
        assert_plan_matches(p, case["expect"], case["name"])


def test_golden_grid_batched(planner):
    """All golden grid cases with equal options in ONE call (segments)."""
    grid = capi.synthetic_grid()
    cases = [c for c in load_golden("grid") if c["stages"] == 4 and not c["encdec"]
             and c["replica_count"] == 1 and c["t_max_interval"] == (5.0).hex() and c["mem_cap"] == "inf"]
    assert len(cases) >= 5
    samples = np.concatenate([np.array(c["samples"], np.int64) for c in cases])
    off = np.concatenate([[0], np.cumsum([c["n"] for c in cases])]).astype(np.int64)
    r = planner.plan_batch(samples, off, grid, capi.Model.uniform(4, 2, False), 4, 1, math.inf, 5.0)
    for s, c in enumerate(cases):
        m = int(r["count"][s])
        got = capi.Plan(int(r["status"][s]), r["splits"][off[s]:off[s] + m], r["mb_times"][off[s]:off[s] + m],
                        float(r["t_max_used"][s]), float(r["objective"][s]), int(r["err_sample_id"][s]),
                        r["ordered"][off[s]:off[s + 1]])
        assert_plan_matches(got, c["expect"], c["name"])


def test_golden_c1(planner):
    case = load_golden("c1")
    cfg = W.CONFIGS["C1"]
    p = planner.plan(W.dataset(cfg, 1), W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
    assert_plan_matches(p, case["expect"], "C1")


def test_golden_c3(planner):
    case = load_golden("c3")
    cfg = W.CONFIGS["C3"]
    p = planner.plan(W.dataset(cfg, 1), W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
    assert_plan_matches(p, case["expect"], "C3")
    assert len(p.splits) == 4168


def test_c2_matches_oracle(planner, orc):
    cfg = W.CONFIGS["C2"]
    s = W.dataset(cfg, 1)
    a = orc.plan(s, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
    b = planner.plan(s, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
    assert_plan_matches(b, record(a), "C2")


def test_c4_subset_matches_oracle(planner, orc):
    cfg = W.CONFIGS["C4"]
    M = 6
    s = W.dataset(cfg, M)
    off = W.seg_offsets(cfg, M)
    r = planner.plan_batch(s, off, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
    for k in (0, 5):
        a = orc.plan(s[off[k]:off[k + 1]], W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
        m = int(r["count"][k])
        got = capi.Plan(int(r["status"][k]), r["splits"][off[k]:off[k] + m], r["mb_times"][off[k]:off[k] + m],
                        float(r["t_max_used"][k]), float(r["objective"][k]), -1,
                        r["ordered"][off[k]:off[k + 1]])
        assert_plan_matches(got, record(a), f"C4[{k}]")


def test_random_grid_vs_oracle(planner, orc):
    grid = capi.synthetic_grid()
    rng = np.random.default_rng(7)
    for k in range(60):
        n = int(rng.integers(1, 300))
        encdec = bool(rng.integers(0, 2))
        C = int(rng.choice([1, 2, 4, 7, 16]))
        L = int(rng.choice([64, 1024, 8192]))
        s = capi.synthetic_dataset(n, L, 900 + k, W.INPUT_DIST, W.T5_TARGET_DIST if encdec else None)
        s[:, 0] = rng.permutation(n) * 3 + 11
        model = capi.Model.uniform(C, int(rng.integers(1, 4)), encdec, recompute=int(rng.integers(0, 3)))
        o = orc.order_samples(s)
        act = max(orc.slice_cost(grid, model, o, i, i + 1)[1] for i in range(n))
        cap = float(rng.choice([math.inf, 1.0 * act, 2.5 * act, 0.9 * act]))
        interval = float(rng.choice([0.0, 5.0, 100.0, 2000.0, 1e5]))
        d = int(rng.integers(1, 3))
        a = orc.plan(s, grid, model, C, d, cap, interval)
        b = _plan_or_status(lambda: planner.plan(s, grid, model, C, d, cap, interval))
        assert_plan_matches(b, record(a), f"random {k}: n={n} C={C} I={interval} cap={cap}")


@pytest.mark.parametrize("name", ["C1", "C3", "C4"])
def test_slice_reuse_matches_per_slice_pricing(name):
    """Pass B's diagonal reuse (band_run_kernel: each distinct (micro-batch
    size, padded length) pair priced once) against pricing every slice
    (band3_kernel): identical plans, candidate counts and slice counts."""
    cfg = W.CONFIGS[name]
    M = {"C1": 64, "C3": 6, "C4": 24}[name]
    s = W.dataset(cfg, M)
    off = W.seg_offsets(cfg, M)
    a = capi.Planner(0)
    b = capi.Planner(0)
    a.set_tuning(slice_table=False)  # the diagonal reuse lives on the band path
    b.set_tuning(slice_reuse=False, slice_table=False)
    ra = a.plan_batch(s, off, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
    rb = b.plan_batch(s, off, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
    for k in ("ordered", "count", "t_max_used", "objective", "status"):
        assert ra[k].tobytes() == rb[k].tobytes(), k
    for q in range(M):
        m = int(ra["count"][q])
        for k in ("splits", "mb_times"):
            assert ra[k][off[q]:off[q] + m].tobytes() == rb[k][off[q]:off[q] + m].tobytes(), (k, q)
    sa, sb = a.stats(), b.stats()
    for k in ("candidates_generated", "candidates_evaluated", "slices_pass_b"):
        assert sa[k] == sb[k], k
    a.close()
    b.close()


@pytest.mark.parametrize("name", ["C1", "C3", "C4"])
def test_band_truncation_matches_full_stream(name):
    """Candidate passes that stop streaming a tile at the first chunk whose
    slices all exceed t (certified monotone slice times on length-sorted
    segments) against streaming every column: identical plans, fewer
    transitions."""
    cfg = W.CONFIGS[name]
    M = {"C1": 64, "C3": 6, "C4": 24}[name]
    s = W.dataset(cfg, M)
    off = W.seg_offsets(cfg, M)
    a = capi.Planner(0)
    b = capi.Planner(0)
    a.set_tuning(slice_table=False)  # the truncation lives on the band path
    b.set_tuning(band_trunc=False, slice_table=False)
    ra = a.plan_batch(s, off, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
    rb = b.plan_batch(s, off, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
    for k in ("ordered", "count", "t_max_used", "objective", "status"):
        assert ra[k].tobytes() == rb[k].tobytes(), k
    for q in range(M):
        m = int(ra["count"][q])
        for k in ("splits", "mb_times"):
            assert ra[k][off[q]:off[q] + m].tobytes() == rb[k][off[q]:off[q] + m].tobytes(), (k, q)
    sa, sb = a.stats(), b.stats()
    assert sa["candidates_evaluated"] == sb["candidates_evaluated"]
    assert sa["transitions_executed"] < sb["transitions_executed"]
    a.close()
    b.close()


@pytest.mark.parametrize("name", ["C1", "C3", "C4"])
def test_slice_table_matches_band(name):
    """The call's shared slice table (gtab.cu: G[length][d] priced once, the
    DP's tiles and the candidate scan read from it) against the per
    mini-batch band of cost pass B: identical plans, candidate sets,
    reference-loop counts and bound transitions; no band written."""
    cfg = W.CONFIGS[name]
    M = {"C1": 64, "C3": 6, "C4": 24}[name]
    s = W.dataset(cfg, M)
    off = W.seg_offsets(cfg, M)
    a = capi.Planner(0)
    b = capi.Planner(0)
    b.set_tuning(slice_table=False, band_trunc=False)  # (the table path streams whole tiles)
    ra = a.plan_batch(s, off, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
    sa = a.stats()
    rb = b.plan_batch(s, off, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
    sb = b.stats()
    assert sa["band_bytes"] == 0 and sb["band_bytes"] > 0
    for k in ("ordered", "count", "t_max_used", "objective", "status"):
        assert ra[k].tobytes() == rb[k].tobytes(), k
    for q in range(M):
        m = int(ra["count"][q])
        for k in ("splits", "mb_times"):
            assert ra[k][off[q]:off[q] + m].tobytes() == rb[k][off[q]:off[q] + m].tobytes(), (k, q)
    for k in ("candidates_generated", "candidates_ref_evaluated", "bound_transitions"):
        assert sa[k] == sb[k], k
    a.close()
    b.close()


@pytest.mark.parametrize("name", ["C1", "C3", "C4", "random"])
def test_bin_intervals_match_row_scan(name):
    """The candidate bins of interval rows (gtab_rowinfo_kernel: two table
    entries per run) against the entry-by-entry scan of the same rows:
    identical plans, candidate sets, reference-loop counts and scanned-entry
    counts (BASELINE configs, and random grids with fine intervals where the
    bins step by more than one and rows fall back to the scan)."""
    cases = []
    if name == "random":
        rng = np.random.default_rng(99)
        for k in range(12):
            M, n = int(rng.integers(1, 6)), int(rng.integers(2, 900))
            s = capi.synthetic_dataset(n * M, int(rng.choice([64, 1024, 8192])), 900 + k, W.INPUT_DIST)
            s[:, 0] = rng.permutation(n * M) + 1
            C = int(rng.choice([2, 4, 16]))
            model = capi.Model.uniform(C, 2, False)
            tot = 1e5 * n
            cases.append((s, np.arange(M + 1, dtype=np.int64) * n, capi.synthetic_grid(), model, C,
                          float(rng.choice([math.inf, 50.0, 400.0])), float(rng.choice([5.0, tot / 64, tot / 4096]))))
    else:
        cfg = W.CONFIGS[name]
        M = {"C1": 64, "C3": 6, "C4": 24}[name]
        cases.append((W.dataset(cfg, M), W.seg_offsets(cfg, M), W.grid(), W.model(cfg), cfg.stages, cfg.mem_cap,
                      cfg.interval))
    a = capi.Planner(0)
    b = capi.Planner(0)
    b.set_tuning(bin_intervals=False)
    for s, off, grid, model, C, cap, interval in cases:
        ra = a.plan_batch(s, off, grid, model, C, 1, cap, interval)
        sa = a.stats()
        rb = b.plan_batch(s, off, grid, model, C, 1, cap, interval)
        sb = b.stats()
        for k in ("ordered", "status", "err_sample_id"):
            assert ra[k].tobytes() == rb[k].tobytes(), k
        for q in range(len(off) - 1):
            if ra["status"][q] != 0:
                continue
            m = int(ra["count"][q])
            for k in ("count", "t_max_used", "objective"):
                assert ra[k][q] == rb[k][q] or (ra[k][q] != ra[k][q] and rb[k][q] != rb[k][q]), (k, q)
            for k in ("splits", "mb_times"):
                assert ra[k][off[q]:off[q] + m].tobytes() == rb[k][off[q]:off[q] + m].tobytes(), (k, q)
        for k in ("candidates_generated", "candidates_ref_evaluated", "slices_pass_b", "bound_transitions"):
            assert sa[k] == sb[k], (k, sa[k], sb[k])
    a.close()
    b.close()


def test_slice_table_random_vs_oracle(orc):
    """The slice-table path on random length-sorted GPT mini-batches
    (duplicate-heavy and distinct lengths, binding and loose caps, several
    intervals, stage counts and recompute strategies, several mini-batches
    per call sharing one table) against the C restatement."""
    grid = capi.synthetic_grid()
    rng = np.random.default_rng(777)
    p = capi.Planner(0)
    for k in range(30):
        M = int(rng.integers(1, 5))
        n = int(rng.integers(1, 600))
        L = int(rng.choice([8, 64, 1024, 8192, 60000]))
        s = capi.synthetic_dataset(n * M, L, 5000 + k, W.INPUT_DIST)
        s[:, 0] = rng.permutation(n * M) + 3
        C = int(rng.choice([2, 4, 16]))
        model = capi.Model.uniform(C, int(rng.integers(1, 4)), False, recompute=int(rng.integers(0, 3)))
        o = orc.order_samples(s[:n])
        act = max(orc.slice_cost(grid, model, o, i, i + 1)[1] for i in range(n))
        cap = float(rng.choice([math.inf, 1.0 * act, 3.0 * act, 40.0 * act]))
        tot = orc.slice_cost(grid, model, o, 0, n)[0]
        interval = float(rng.choice([5.0, tot / 7.0, tot / 64.0, tot / 300.0]))
        off = np.arange(M + 1, dtype=np.int64) * n
        r = p.plan_batch(s, off, grid, model, C, 1, cap, interval)
        for q in range(M):
            a = orc.plan(s[off[q]:off[q + 1]], grid, model, C, 1, cap, interval)
            m = int(r["count"][q])
            got = capi.Plan(int(r["status"][q]), r["splits"][off[q]:off[q] + m], r["mb_times"][off[q]:off[q] + m],
                            float(r["t_max_used"][q]), float(r["objective"][q]), int(r["err_sample_id"][q]),
                            r["ordered"][off[q]:off[q + 1]])
            assert_plan_matches(got, record(a), f"table {k}.{q}: n={n} C={C} I={interval} cap={cap}")
    p.close()


def test_band_path_random_capped_vs_oracle(orc):
    """The band path (cost pass B writes per mini-batch tiles, the DP streams
    them with TMA) on random GPT mini-batches (binding and non-binding caps,
    duplicate-heavy and distinct lengths, ragged last blocks, several
    intervals and stage counts) against the C restatement."""
    grid = capi.synthetic_grid()
    rng = np.random.default_rng(4242)
    priced = capi.Planner(0)
    priced.set_tuning(slice_table=False)
    for k in range(40):
        n = int(rng.integers(1, 700))
        L = int(rng.choice([8, 64, 1024, 8192]))
        s = capi.synthetic_dataset(n, L, 3000 + k, W.INPUT_DIST)
        s[:, 0] = rng.permutation(n) + 7
        C = int(rng.choice([2, 4, 16]))
        model = capi.Model.uniform(C, int(rng.integers(1, 4)), False, recompute=int(rng.integers(0, 3)))
        o = orc.order_samples(s)
        act = max(orc.slice_cost(grid, model, o, i, i + 1)[1] for i in range(n))
        cap = float(rng.choice([math.inf, 1.0 * act, 3.0 * act, 40.0 * act]))
        tot = orc.slice_cost(grid, model, o, 0, n)[0]
        interval = float(rng.choice([5.0, tot / 7.0, tot / 64.0, tot / 300.0]))
        a = orc.plan(s, grid, model, C, 1, cap, interval)
        b = _plan_or_status(lambda: priced.plan(s, grid, model, C, 1, cap, interval))
        assert_plan_matches(b, record(a), f"band {k}: n={n} C={C} I={interval} cap={cap}")
    priced.close()


@pytest.mark.parametrize("slice_table", [True, False])
def test_global_state_dp_vs_streaming_oracle(orc, slice_table):
    """Uncapped 10,000-sample GPT mini-batches: the DP state (20 B x ~10k
    rows) no longer fits shared memory, so the passes keep it in an
    L2-resident global array — on the slice-table and the band path —
    against the streaming C restatement (O(n) memory)."""
    grid = capi.synthetic_grid()
    p = capi.Planner(0)
    p.set_tuning(slice_table=slice_table)
    for k, n in enumerate((10000, 9985)):  # (a ragged last block)
        s = capi.synthetic_dataset(n, 8192, 900 + k, W.INPUT_DIST)
        model = capi.Model.uniform(4, 2, False)
        tot = orc.slice_cost(grid, model, orc.order_samples(s), 0, n)[0]
        interval = tot / 40.0
        a = orc.plan_stream(s, grid, model, 4, 1, math.inf, interval)
        b = p.plan(s, grid, model, 4, 1, math.inf, interval)
        assert_plan_matches(b, record(a), f"global state n={n} table={slice_table}")
    p.close()


def test_slice_reuse_duplicate_heavy_vs_oracle(planner, orc):
    """Few distinct lengths (long runs), ragged sizes, binding and loose caps,
    fine and coarse intervals: the reuse path against the C restatement."""
    grid = capi.synthetic_grid()
    rng = np.random.default_rng(23)
    for k in range(40):
        n = int(rng.integers(1, 1500))
        distinct = int(rng.choice([1, 2, 5, 30, 200]))
        vals = rng.choice(np.arange(1, 4097), size=distinct, replace=False)
        s = np.zeros((n, 3), np.int64)
        s[:, 0] = rng.permutation(n) * 5 + 3
        s[:, 1] = rng.choice(vals, size=n)
        C = int(rng.choice([1, 4, 16]))
        model = capi.Model.uniform(C, int(rng.integers(1, 4)), False, recompute=int(rng.integers(0, 3)))
        o = orc.order_samples(s)
        act = max(orc.slice_cost(grid, model, o, i, i + 1)[1] for i in range(0, n, max(1, n // 50)))
        act = max(act, orc.slice_cost(grid, model, o, n - 1, n)[1])
        cap = float(rng.choice([math.inf, 1.0 * act, 3.0 * act, 20.0 * act]))
        interval = float(rng.choice([1.0, 50.0, 1000.0, 1e5]))
        a = orc.plan(s, grid, model, C, 1, cap, interval)
        b = _plan_or_status(lambda: planner.plan(s, grid, model, C, 1, cap, interval))
        assert_plan_matches(b, record(a), f"dup-heavy {k}: n={n} distinct={distinct} C={C} I={interval}")


def test_random_tables_vs_oracle(planner, orc):
    """Generic SliceCostFn path with non-monotone, tie-heavy and negative costs."""
    rng = np.random.default_rng(11)
    for k in range(80):
        n = int(rng.integers(1, 60))
        tri = n * (n + 1) // 2
        kind = k % 4
        if kind == 0:
            T = rng.integers(0, 5, tri).astype(float)         # many ties
        elif kind == 1:
            T = rng.random(tri) * 100.0                       # non-monotone
        elif kind == 2:
            T = rng.integers(-3, 10, tri).astype(float)       # negative times
        else:
            T = np.round(rng.random(tri) * 20.0, 1)
        M = rng.random(tri) * 10.0
        cap = float(rng.choice([math.inf, 5.0, 9.0]))
        # keep singletons feasible most of the time
        idx = 0
        for i in range(n):
            if rng.random() < 0.97:
                M[idx] = min(M[idx], 1.0)
            idx += n - i
        C = int(rng.choice([1, 2, 3, 6]))
        d = int(rng.integers(1, 3))
        interval = float(rng.choice([0.0, 0.5, 3.0]))
        a = orc.plan_tables(T, M, n, C, d, cap, interval)
        b = _plan_or_status(lambda: planner.plan_tables(T, M, n, C, d, cap, interval))
        if a.status == 2:  # plan_tables reports the ordered index
            assert b.status == 2 and b.err_sample_id == a.err_sample_id, k
            continue
        assert_plan_matches(b, record(a, False), f"tables {k}")


def test_sort_matches_oracle(planner, orc):
    rng = np.random.default_rng(3)
    for k in range(12):
        n = int(rng.integers(1, 20000))
        s = np.stack([rng.permutation(n), rng.integers(1, 9000, n), rng.integers(0, 300, n)], 1)
        if k % 3 == 1:  # wide fields -> three-word key path
            s[:, 0] = rng.integers(-(1 << 62), 1 << 62, n)
            s[:, 1] = rng.integers(-(1 << 40), 1 << 40, n)
        assert np.array_equal(planner.order_samples(s), orc.order_samples(s)), k
    # segmented: many segments in one call
    s = np.stack([np.arange(5000), rng.integers(1, 100, 5000), rng.integers(0, 3, 5000)], 1)
    off = np.array([0, 1, 2, 500, 501, 4000, 5000], np.int64)
    got = planner.order_samples(s, off)
    for a, b in zip(off[:-1], off[1:]):
        assert np.array_equal(got[a:b], orc.order_samples(s[a:b]))


def test_invalid_arguments(planner):
    grid = capi.synthetic_grid()
    model = capi.Model.uniform(2, 2, False)
    s = capi.synthetic_dataset(10, 100, 1)
    with pytest.raises(capi.InvalidArgument):
        planner.plan(s, grid, model, 0)
    with pytest.raises(capi.InvalidArgument):
        planner.plan(s, grid, model, 2, 0)
    with pytest.raises(capi.InvalidArgument):
        planner.plan(s, grid, model, 2, 1, math.inf, -1.0)
    with pytest.raises(capi.InvalidArgument):
        planner.plan_tables(np.zeros(0), np.zeros(0), 0, 2)


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not shipped")
def test_random_vs_reference(planner):
    ref = Reference()
    grid = capi.synthetic_grid()
    rng = np.random.default_rng(21)
    for k in range(15):
        n = int(rng.integers(2, 400))
        encdec = bool(k % 2)
        s = capi.synthetic_dataset(n, 8192, 40 + k, W.INPUT_DIST, W.T5_TARGET_DIST if encdec else None)
        model = capi.Model.uniform(4, 2, encdec)
        a = ref.plan(s, grid, model, 4, 1, math.inf, 5000.0)
        b = planner.plan(s, grid, model, 4, 1, math.inf, 5000.0)
        assert_plan_matches(b, record(a), f"ref {k}")


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not shipped")
def test_nan_interval_plans_like_the_reference(planner):
    """A NaN t_max_interval is accepted by the reference (microbatch.cpp:225
    tests `< 0`) and selects the exact candidate set (`> 0` at :263)."""
    ref = Reference()
    grid = capi.synthetic_grid()
    for encdec in (False, True):
        s = capi.synthetic_dataset(300, 8192, 77, W.INPUT_DIST, W.T5_TARGET_DIST if encdec else None)
        model = capi.Model.uniform(4, 2, encdec)
        a = ref.plan(s, grid, model, 4, 1, math.inf, math.nan)
        b = planner.plan(s, grid, model, 4, 1, math.inf, math.nan)
        assert_plan_matches(b, record(a), f"nan interval encdec={encdec}")
        c = planner.plan(s, grid, model, 4, 1, math.inf, 0.0)
        assert c.splits.tobytes() == b.splits.tobytes() and c.t_max_used == b.t_max_used


def _monotone_grid(rng, nm=5, ns=6, jitter=False):
    """Random grid whose cells grow along both axes (cumulative sums of
    positive steps); jitter=True breaks monotonicity of act_mem."""
    mbs = np.cumsum(rng.integers(1, 4, nm)).astype(np.int64)
    mbs[0] = 1
    seq = np.cumsum(rng.integers(8, 200, ns)).astype(np.int64)
    cells = np.zeros((2, 3, nm, ns, 3))
    for k in range(2):
        for r in range(3):
            for f in range(3):
                step = rng.random((nm, ns)) * 3.0 + 0.01
                cells[k, r, :, :, f] = np.cumsum(np.cumsum(step, 0), 1)
    if jitter:
        cells[:, :, nm // 2, ns // 2, 2] *= 0.2  # a dip in act_mem
    return capi.Grid(mbs, seq, cells)


def test_pass_a_certificate_engaged_c3(planner):
    """C3 (binding cap): the certified row exit prices ~the band only, and
    the batched result still equals the reference's golden plan."""
    case = load_golden("c3")
    cfg = W.CONFIGS["C3"]
    M = 3
    r = planner.plan_batch(W.dataset(cfg, M), W.seg_offsets(cfg, M), W.grid(), W.model(cfg), cfg.stages,
                           1, cfg.mem_cap, cfg.interval)
    st = planner.stats()
    assert math.isfinite(st["exit_thresh"]) and st["exit_thresh"] > cfg.mem_cap
    assert st["exit_thresh"] - cfg.mem_cap < 1e-6 * cfg.mem_cap
    full = M * cfg.n * (cfg.n + 1) // 2
    assert st["slices_pass_a"] < full // 5, (st["slices_pass_a"], full)
    m = int(r["count"][0])
    got = capi.Plan(int(r["status"][0]), r["splits"][:m], r["mb_times"][:m], float(r["t_max_used"][0]),
                    float(r["objective"][0]), -1, r["ordered"][:cfg.n])
    assert_plan_matches(got, case["expect"], "C3 batched")


@pytest.mark.parametrize("jitter", [False, True])
def test_pass_a_certificate_random_grids(planner, orc, jitter):
    rng = np.random.default_rng(5 + jitter)
    for k in range(12):
        grid = _monotone_grid(rng, jitter=jitter)
        n = int(rng.integers(20, 400))
        encdec = bool(k % 2)
        s = capi.synthetic_dataset(n, int(rng.choice([300, 2000])), 70 + k, W.INPUT_DIST,
                                   W.T5_TARGET_DIST if encdec else None)
        model = capi.Model.uniform(int(rng.choice([2, 4])), 2, encdec)
        o = orc.order_samples(s)
        acts = [orc.slice_cost(grid, model, o, i, i + 1)[1] for i in range(n)]
        cap = float(max(acts) * rng.choice([1.0, 1.7, 3.0]))
        interval = float(rng.choice([0.0, 5.0, 50.0]))
        a = orc.plan(s, grid, model, model.encoder_layers.size, 1, cap, interval)
        b = _plan_or_status(lambda: planner.plan(s, grid, model, model.encoder_layers.size, 1, cap, interval))
        st = planner.stats()
        if jitter:
            assert math.isinf(st["exit_thresh"]), k  # no certificate: full scan
        assert_plan_matches(b, record(a), f"cert grid {k} jitter={jitter}")


@pytest.mark.parametrize("bad", [math.inf, math.nan])
def test_nonfinite_grid_cells_match_oracle(planner, orc, bad):
    """The reference accepts any non-negative cells (cost_model.cpp:86-88; NaN
    and +inf pass its check).  Blends through such cells produce NaN, which
    std::max(0.0, v) maps to 0.0 (cost_model.cpp:141) — the device must clamp
    exactly the same way."""
    g = capi.synthetic_grid()
    cells = g.cells.copy()
    cells[:, :, 3, 4, :] = bad
    cells[1, 0, 6, 2, 0] = bad
    grid = capi.Grid(g.mbs_axis, g.seq_axis, cells)
    rng = np.random.default_rng(17)
    for k in range(8):
        n = int(rng.integers(5, 200))
        encdec = bool(k % 2)
        s = capi.synthetic_dataset(n, 4096, 300 + k, W.INPUT_DIST, W.T5_TARGET_DIST if encdec else None)
        model = capi.Model.uniform(4, 2, encdec)
        interval = float(rng.choice([0.0, 50.0, 5000.0]))
        a = orc.plan(s, grid, model, 4, 1, math.inf, interval)
        b = _plan_or_status(lambda: planner.plan(s, grid, model, 4, 1, math.inf, interval))
        assert_plan_matches(b, record(a), f"nonfinite {bad} {k}")


def test_concurrent_sub_batches_match_single_stream():
    """pp_tuning::streams splits a batch over concurrent sub-contexts; the
    plans must be identical to the single-stream call (and the golden C3)."""
    cfg = W.CONFIGS["C3"]
    M = 7
    s = W.dataset(cfg, M)
    off = W.seg_offsets(cfg, M)
    a = capi.Planner(0)
    b = capi.Planner(0)
    b.set_tuning(streams=3)
    ra = a.plan_batch(s, off, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
    rb = b.plan_batch(s, off, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
    for k in ("ordered", "count", "t_max_used", "objective", "status"):
        assert ra[k].tobytes() == rb[k].tobytes(), k
    for q in range(M):  # only the first count[q] entries of a segment are defined
        m = int(ra["count"][q])
        for k in ("splits", "mb_times"):
            assert ra[k][off[q]:off[q] + m].tobytes() == rb[k][off[q]:off[q] + m].tobytes(), (k, q)
    st = b.stats()
    assert st["candidates_evaluated"] == M
    case = load_golden("c3")
    m = int(rb["count"][0])
    got = capi.Plan(int(rb["status"][0]), rb["splits"][:m], rb["mb_times"][:m], float(rb["t_max_used"][0]),
                    float(rb["objective"][0]), -1, rb["ordered"][:cfg.n])
    assert_plan_matches(got, case["expect"], "C3 split")
    a.close()
    b.close()


def test_threads_with_own_contexts_mixed_sizes():
    """Many host threads, one context each, planning small and large
    mini-batches at once (the reference's run_plan pool, driver.cpp:222-242):
    every plan equals the single-threaded one.  Regression: per-launch
    shared-memory limits set by one thread used to fail another thread's
    larger launch in flight."""
    import threading

    cfg = W.CONFIGS["C3"]
    big = W.dataset(cfg, 1)
    grid, model = W.grid(), W.model(cfg)
    rng = np.random.default_rng(5)
    smalls = [big[rng.choice(len(big), int(k), replace=False)] for k in rng.integers(8, 600, 6)]
    jobs = [big] + smalls
    ref_p = capi.Planner(0)
    want = [record(ref_p.plan(s, grid, model, cfg.stages, 1, cfg.mem_cap, cfg.interval)) for s in jobs]
    ref_p.close()
    errors = []

    def worker(t):
        p = capi.Planner(0)
        try:
            for it in range(6):
                k = (t + it) % len(jobs)
                got = p.plan(jobs[k], grid, model, cfg.stages, 1, cfg.mem_cap, cfg.interval)
                assert_plan_matches(got, want[k], f"thread {t} job {k}")
        except BaseException as e:  # noqa: BLE001 - surfaced below
            errors.append(e)
        finally:
            p.close()

    ts = [threading.Thread(target=worker, args=(t,)) for t in range(6)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors[0]


def test_order_output_matches_ordered_samples(planner):
    """pp_plan_out.order (per-segment sample indices) is the ordering the
    `ordered` records carry, for sorted, split-stream and presorted calls."""
    cfg = W.CONFIGS["C3"]
    M = 5
    s = W.dataset(cfg, M)
    off = W.seg_offsets(cfg, M)
    for streams, presorted in ((1, False), (3, False), (1, True)):
        p = capi.Planner(0)
        p.set_tuning(streams=streams)
        a = p.plan_batch(s, off, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval,
                         presorted=presorted)
        b = p.plan_batch(s, off, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval,
                         presorted=presorted, out=capi.Planner.plan_buffers(len(s), M, order_only=True))
        for q in range(M):
            seg = s[off[q]:off[q + 1]]
            assert np.array_equal(seg[b["order"][off[q]:off[q + 1]]], a["ordered"][off[q]:off[q + 1]]), q
            m = int(a["count"][q])
            assert np.array_equal(a["splits"][off[q]:off[q] + m], b["splits"][off[q]:off[q] + m])
        p.close()


def test_pinned_outputs_match_pageable(planner):
    """Pinned output buffers take the valid prefix of splits / mb_times
    through their device alias (prefix_out_kernel) instead of full-length
    copies: same plans as pageable buffers on every host-buffer path
    (single call, part pipeline with 1 and 2 parts per worker, the
    concurrent-worker pipeline), and nothing past count[s] is written."""
    import torch

    def pinned_alloc(shape, dtype):
        t = torch.full(shape if isinstance(shape, tuple) else (shape,), -7,
                       dtype={np.int64: torch.int64, np.int32: torch.int32, np.float64: torch.float64}[dtype])
        return t.pin_memory().numpy()

    cfg = W.CONFIGS["C3"]
    M = 7
    s = W.dataset(cfg, M)
    off = W.seg_offsets(cfg, M)
    for streams, chunks in ((1, 0), (3, 0), (3, 2), (3, -1)):
        p = capi.Planner(0)
        p.set_tuning(streams=streams, host_chunks=chunks)
        a = p.plan_batch(s, off, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
        keep = []

        def alloc(shape, dtype):
            x = pinned_alloc(shape, dtype)
            keep.append(x)
            return x

        b = p.plan_batch(s, off, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval,
                         out=capi.Planner.plan_buffers(len(s), M, alloc, order_only=True))
        for k in ("count", "status", "t_max_used", "objective"):
            assert np.array_equal(a[k].view(np.int64) if a[k].dtype == np.float64 else a[k],
                                  b[k].view(np.int64) if b[k].dtype == np.float64 else b[k]), (streams, chunks, k)
        for q in range(M):
            m = int(a["count"][q])
            lo, hi = off[q], off[q + 1]
            assert np.array_equal(a["splits"][lo:lo + m], b["splits"][lo:lo + m]), (streams, chunks, q)
            assert np.array_equal(a["mb_times"][lo:lo + m].view(np.int64), b["mb_times"][lo:lo + m].view(np.int64))
            if streams > 1:  # the prefix writes leave the rest of the caller's buffer alone
                assert (b["splits"][lo + m:hi] == -7).all(), (streams, chunks, q)
        p.close()


def test_presorted_arbitrary_order_matches_oracle(planner, orc):
    """dp_partition(span) on the caller's order (no sort): running maxima of
    the padded lengths over unsorted spans, certified scan (no bisection)."""
    grid = capi.synthetic_grid()
    rng = np.random.default_rng(31)
    for k in range(10):
        n = int(rng.integers(2, 600))
        encdec = bool(k % 2)
        s = capi.synthetic_dataset(n, 8192, 500 + k, W.INPUT_DIST, W.T5_TARGET_DIST if encdec else None)
        s = s[rng.permutation(n)]
        model = capi.Model.uniform(4, 2, encdec)
        acts = [orc.slice_cost(grid, model, s, i, i + 1)[1] for i in range(n)]
        cap = float(rng.choice([math.inf, 3.0 * max(acts)]))
        interval = float(rng.choice([0.0, 1000.0, 50000.0]))
        a = orc.plan(s, grid, model, 4, 1, cap, interval, presorted=True)
        b = _plan_or_status(lambda: planner.plan(s, grid, model, 4, 1, cap, interval, presorted=True))
        assert_plan_matches(b, record(a), f"presorted {k}")


def test_exact_candidate_set_c2_scale(planner, orc):
    """t_max_interval = 0 (the exact candidate set: segmented u64 sort +
    unique of every feasible slice time) on a BASELINE-C2-sized T5 batch."""
    cfg = W.CONFIGS["C2"]
    s = W.dataset(cfg, 1)
    a = orc.plan(s, W.grid(), W.model(cfg), cfg.stages, 1, math.inf, 0.0)
    b = planner.plan(s, W.grid(), W.model(cfg), cfg.stages, 1, math.inf, 0.0)
    assert_plan_matches(b, record(a), "C2 exact")


def test_replicas_and_capped_t5(planner, orc):
    """D > 1 (balance_replicas on the host, bound / objective divided by D)
    and a binding cap on an encoder-decoder model (scan pass A, target
    running maxima)."""
    grid = capi.synthetic_grid()
    rng = np.random.default_rng(41)
    for k in range(6):
        n = int(rng.integers(50, 900))
        s = capi.synthetic_dataset(n, 8192, 600 + k, W.INPUT_DIST, W.T5_TARGET_DIST)
        model = capi.Model.uniform(8, 2, True)
        o = orc.order_samples(s)
        acts = [orc.slice_cost(grid, model, o, i, i + 1)[1] for i in range(n)]
        cap = float(max(acts) * rng.choice([1.5, 4.0]))
        d = int(rng.integers(2, 5))
        interval = float(rng.choice([0.0, 2000.0]))
        a = orc.plan(s, grid, model, 8, d, cap, interval)
        b = _plan_or_status(lambda: planner.plan(s, grid, model, 8, d, cap, interval))
        assert_plan_matches(b, record(a), f"D={d} T5 cap {k}")


def test_candidate_bins_past_the_threshold_table(planner, orc):
    """Slice times far beyond the 256 binned candidates (I = 5, the paper's
    interval): every bin past the threshold table takes the exact-division
    path; batches of heavy-tailed lengths up to 8192 tokens."""
    grid = capi.synthetic_grid()
    for k, L in enumerate([512, 8192]):
        s = capi.synthetic_dataset(700, L, 77 + k, (capi.LOGNORMAL, 4.0, 2.0, 1, 1, 0.8))
        model = capi.Model.uniform(4, 2, False)
        a = orc.plan(s, grid, model, 4, 1, math.inf, 5.0)
        b = planner.plan(s, grid, model, 4, 1, math.inf, 5.0)
        assert_plan_matches(b, record(a), f"I=5 L={L}")


def test_cooperative_dp_pass_matches_oracle(orc):
    """The whole-GPU cooperative DP pass (dp_coop.cu, used for very long
    mini-batches such as C5), forced onto small mini-batches with
    coop_min_n, against the C restatement: capped and uncapped, GPT and T5,
    quantised and exact candidate sets, and the table path."""
    p = capi.Planner(0)
    p.set_tuning(coop_min_n=1)
    grid = capi.synthetic_grid()
    rng = np.random.default_rng(57)
    for k in range(8):
        n = int(rng.integers(40, 700))
        encdec = bool(k % 2)
        s = capi.synthetic_dataset(n, 8192, 800 + k, W.INPUT_DIST, W.T5_TARGET_DIST if encdec else None)
        model = capi.Model.uniform(4, 2, encdec)
        o = orc.order_samples(s)
        acts = [orc.slice_cost(grid, model, o, i, i + 1)[1] for i in range(n)]
        cap = float(rng.choice([math.inf, 3.0 * max(acts)]))
        interval = float(rng.choice([0.0, 500.0, 20000.0]))
        a = orc.plan(s, grid, model, 4, 1, cap, interval)
        b = _plan_or_status(lambda: p.plan(s, grid, model, 4, 1, cap, interval))
        assert_plan_matches(b, record(a), f"coop {k}")
    for case in load_golden("toy")[:40]:
        T, M = toy_tables(case["lens"], case["mem_per_sample"], case["heavy"])
        got = _plan_or_status(lambda: p.plan_tables(
            T, M, len(case["lens"]), case["stage_count"], case["replica_count"],
            unhex(case["mem_cap"]), unhex(case["t_max_interval"])))
        assert_plan_matches(got, case["expect"], "coop " + case["name"])
    p.close()


@pytest.mark.timeout(900)
def test_c5_long_tail_full_scale():
    """BASELINE config C5 (65,536 T5 sequences up to 65,536 tokens, no cap,
    256 candidates) at full scale — the reference needs ~9 h and 34 GB of
    tables, so the checker is the STREAMING restatement (oracle/pp_stream.c,
    pinned against the unmodified reference at n <= 2048 by
    tests/test_oracle.py), whose output is tests/golden/c5.json: splits,
    slice times (sha256 of the bytes), t_max_used and objective (hex), the
    ordering (sha256 of the ids) and the candidate counters.  Also the
    whole-GPU cooperative DP against the one-CTA DP kernel, bit for bit."""
    import hashlib

    cfg = W.CONFIGS["C5"]
    e = load_golden("c5")["expect"]
    s = W.dataset(cfg, 1)
    coop = capi.Planner(0)
    single = capi.Planner(0)
    single.set_tuning(coop_min_n=1 << 30)  # never cooperative
    a = coop.plan(s, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
    assert len(a.splits) == e["count"]
    assert [int(x) for x in np.diff(np.concatenate([[0], a.splits]))] == e["split_deltas"]
    assert hashlib.sha256(np.ascontiguousarray(a.mb_times, "<f8").tobytes()).hexdigest() == e["mb_times_sha256"]
    assert [float(x).hex() for x in a.mb_times[:8]] == e["mb_time_first"]
    assert float(a.t_max_used).hex() == e["t_max_used"]
    assert float(a.objective).hex() == e["objective"]
    assert hashlib.sha256(np.ascontiguousarray(a.ordered[:, 0], "<i8").tobytes()).hexdigest() == \
        e["ordered_ids_sha256"]
    assert (a.n_candidates, a.n_evaluated) == (e["n_candidates"], e["n_evaluated"])
    b = single.plan(s, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
    assert np.array_equal(a.splits, b.splits)
    assert a.mb_times.tobytes() == b.mb_times.tobytes()
    assert a.t_max_used == b.t_max_used and a.objective == b.objective
    coop.close()
    single.close()


@pytest.mark.timeout(900)
@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not shipped")
def test_c4_64_minibatches_match_reference(planner):
    """BASELINE config C4's epoch shape: 64 consecutive 2048-seq mini-batches
    planned in ONE device call, against the unmodified reference planning the
    same mini-batches on every host core (run_plan's pool): every plan's
    splits, slice times, ordering, t_max_used and objective bit for bit."""
    import os

    cfg = W.CONFIGS["C4"]
    M = 64
    s = W.dataset(cfg, M)
    off = W.seg_offsets(cfg, M)
    r = planner.plan_batch(s, off, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
    ref = Reference().plan_batch_full(s, off, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap,
                                      cfg.interval, threads=os.cpu_count() or 1)
    assert np.array_equal(ref["status"], r["status"]) and np.all(r["status"] == 0)
    assert np.array_equal(ref["count"], r["count"])
    assert ref["t_max_used"].tobytes() == r["t_max_used"].tobytes()
    assert ref["objective"].tobytes() == r["objective"].tobytes()
    assert np.array_equal(ref["ordered_ids"], r["ordered"][:, 0])
    for k in range(M):
        m = int(r["count"][k])
        sl = slice(off[k], off[k] + m)
        assert np.array_equal(ref["splits"][sl], r["splits"][sl]), f"C4[{k}] splits"
        assert ref["mb_times"][sl].tobytes() == r["mb_times"][sl].tobytes(), f"C4[{k}] times"


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not shipped")
def test_op_cost_tables_match_reference(planner):
    """OpCostTable::from_shapes on the device against
    the unmodified reference's from_shapes: every recompute strategy, GPT and
    T5 layouts, shapes inside, below and beyond the grid axes."""
    ref = Reference()
    grid = capi.synthetic_grid()
    rng = np.random.default_rng(63)
    for encdec in (False, True):
        for r in range(3):
            model = capi.Model.uniform(int(rng.choice([1, 4, 8])), int(rng.integers(1, 4)), encdec, recompute=r)
            sh = np.stack([rng.integers(1, 600, 400), rng.integers(0, 90000, 400),
                           rng.integers(0, 9000, 400)], 1)
            a = ref.op_costs(sh, grid, model)
            b = planner.op_costs(sh, grid, model)
            for x, y, nm in zip(a, b, ("t_f", "t_b", "act_mem")):
                assert x.tobytes() == y.tobytes(), (nm, encdec, r)


def test_plan_op_costs_device_match_reference_shapes(planner):
    """Op-cost tables of device-resident C3 plans (padded shape of every planned
    micro-batch) equal the reference's from_shapes over the same shapes."""
    import torch

    cfg = W.CONFIGS["C3"]
    M = 3
    s = W.dataset(cfg, M)
    off = W.seg_offsets(cfg, M)
    d_s = torch.from_numpy(s).cuda()
    d_off = torch.from_numpy(off).cuda()
    tot = M * cfg.n
    out = {"ordered": torch.empty((tot, 3), dtype=torch.int64, device="cuda"),
           "splits": torch.empty(tot, dtype=torch.int32, device="cuda"),
           "mb_times": torch.empty(tot, dtype=torch.float64, device="cuda"),
           "count": torch.empty(M, dtype=torch.int32, device="cuda"),
           "t_max_used": torch.empty(M, dtype=torch.float64, device="cuda"),
           "objective": torch.empty(M, dtype=torch.float64, device="cuda"),
           "status": torch.empty(M, dtype=torch.int32, device="cuda"),
           "err_sample_id": torch.empty(M, dtype=torch.int64, device="cuda")}
    planner.plan_batch_device(d_s, d_off, off, out, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap,
                              cfg.interval)
    C_ = cfg.stages
    cap = tot
    tf, tb, act = (torch.empty(cap * C_, dtype=torch.float64, device="cuda") for _ in range(3))
    model = capi.Model.uniform(cfg.stages, 2, False, recompute=2)  # a replica may price another strategy
    mb_off = planner.plan_op_costs_device(out["ordered"], d_off, off, out["splits"], out["count"],
                                          W.grid(), model, tf, tb, act)
    ordered = out["ordered"].cpu().numpy()
    splits = out["splits"].cpu().numpy()
    count = out["count"].cpu().numpy()
    shapes = []
    for q in range(M):
        sp = splits[off[q]:off[q] + count[q]]
        lo = 0
        for e in sp:
            blk = ordered[off[q] + lo:off[q] + e]
            shapes.append((e - lo, max(0, blk[:, 1].max()), max(0, blk[:, 2].max())))
            lo = e
    assert mb_off[-1] == len(shapes)
    host = planner.op_costs(np.array(shapes, np.int64), W.grid(), model)
    n_mb = len(shapes)
    for x, y in zip(host, (tf, tb, act)):
        assert x.reshape(-1).tobytes() == y[:n_mb * C_].cpu().numpy().tobytes()
    if reference_available():
        ref = Reference().op_costs(np.array(shapes, np.int64), W.grid(), model)
        assert ref[0].tobytes() == host[0].tobytes() and ref[2].tobytes() == host[2].tobytes()


def _recompute_cases(rng, grid, model, orc_act):
    """(shapes, mb_offset, limits, strategies) cases around the strategies'
    activation maxima: every strategy fits, only Selective / Full fit, none
    fits, limits on the boundary (act == limit violates), empty partitions,
    restricted strategy sets."""
    cases = []
    for k in range(16):
        S = int(rng.integers(1, 7))
        counts = rng.integers(0 if k % 5 == 0 else 1, 40, S)
        off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        n = int(off[-1])
        sh = np.stack([rng.integers(1, 300, n), rng.integers(0, 9000, n), rng.integers(0, 700, n)], 1).astype(np.int64)
        acts = [orc_act(sh, r) for r in range(3)]  # per strategy (n, C) tables
        C_ = len(model.encoder_layers)
        mx = [a.max(0) if len(a) else np.zeros(C_) for a in acts]
        pick = k % 4
        if pick == 0:
            lim = mx[0] * 1.01 + 1.0           # everything fits: None
        elif pick == 1:
            lim = (mx[0] + mx[1]) / 2          # None violates somewhere, Selective may fit
        elif pick == 2:
            lim = np.minimum(mx[2], mx[1]) * 0.5  # nothing fits: the last strategy's stage
        else:
            lim = mx[1].copy()                 # boundary: act == limit violates
        strategies = [(0, 1, 2), (2,), (1, 2), (0, 2)][k % 4]
        cases.append((sh, off, np.ascontiguousarray(lim, np.float64), strategies))
    return cases


def test_select_recomputation_matches_reference(planner):
    """pp_select_recomputation (schedule.cpp:319-364)
    against the reference's select_recomputation on the same shapes: chosen
    strategy, InfeasibleError stage, and the chosen tables bit for bit
    (GPT and T5, 4 and 8 stages)."""
    if not reference_available():
        pytest.skip("oracle/_ref not built")
    ref = Reference()
    rng = np.random.default_rng(31)
    grid = W.grid()
    for C_, encdec in ((4, False), (8, True)):
        model = capi.Model.uniform(C_, 2, encdec)

        def orc_act(sh, r):
            m = capi.Model.uniform(C_, 2, encdec, recompute=r)
            return planner.op_costs(sh, grid, m)[2] if len(sh) else np.zeros((0, C_))

        for sh, off, lim, strat in _recompute_cases(rng, grid, model, orc_act):
            got = planner.select_recomputation(sh, off, grid, model, strat, lim)
            exp = ref.select_recomputation(sh, off, grid, model, strat, lim)
            assert got["strategy"].tolist() == exp["strategy"].tolist(), (strat, got["strategy"], exp["strategy"])
            assert got["violating_stage"].tolist() == exp["violating_stage"].tolist()
            for q in range(len(off) - 1):
                if exp["strategy"][q] < 0:
                    continue
                a, b = off[q], off[q + 1]
                for k in ("t_f", "t_b", "act_mem"):
                    assert got[k][a:b].tobytes() == exp[k][a:b].tobytes(), (k, q)
    with pytest.raises(capi.InvalidArgument):
        planner.select_recomputation(sh, off, grid, model, (), lim)


def test_select_recomputation_device_plans(planner):
    """select_recomputation over device-resident C1 plans (the padded shape of
    each planned micro-batch) equals the host entry point on those shapes;
    limits make some mini-batches take Selective / Full."""
    import torch

    cfg = W.CONFIGS["C1"]
    M = 48
    s = W.dataset(cfg, M)
    off = W.seg_offsets(cfg, M)
    d_s, d_off = torch.from_numpy(s).cuda(), torch.from_numpy(off).cuda()
    tot = M * cfg.n
    out = {"ordered": torch.empty((tot, 3), dtype=torch.int64, device="cuda"),
           "splits": torch.empty(tot, dtype=torch.int32, device="cuda"),
           "mb_times": torch.empty(tot, dtype=torch.float64, device="cuda"),
           "count": torch.empty(M, dtype=torch.int32, device="cuda"),
           "t_max_used": torch.empty(M, dtype=torch.float64, device="cuda"),
           "objective": torch.empty(M, dtype=torch.float64, device="cuda"),
           "status": torch.empty(M, dtype=torch.int32, device="cuda"),
           "err_sample_id": torch.empty(M, dtype=torch.int64, device="cuda")}
    planner.plan_batch_device(d_s, d_off, off, out, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap,
                              cfg.interval)
    C_ = cfg.stages
    model = W.model(cfg)
    ordered, splits, count = (out[k].cpu().numpy() for k in ("ordered", "splits", "count"))
    shapes, mbo = [], [0]
    for q in range(M):
        lo = 0
        for e in splits[off[q]:off[q] + count[q]]:
            blk = ordered[off[q] + lo:off[q] + e]
            shapes.append((e - lo, max(0, blk[:, 1].max()), max(0, blk[:, 2].max())))
            lo = e
        mbo.append(len(shapes))
    shapes = np.array(shapes, np.int64)
    act0 = planner.op_costs(shapes, W.grid(), model)[2]
    lim = np.quantile(act0, 0.9, axis=0)  # the heaviest mini-batches must recompute
    tf, tb, act = (torch.empty(len(shapes) * C_, dtype=torch.float64, device="cuda") for _ in range(3))
    st, vs = (torch.empty(M, dtype=torch.int32, device="cuda") for _ in range(2))
    mb_off = planner.select_recomputation_device(out["ordered"], d_off, off, out["splits"], out["count"],
                                                 W.grid(), model, lim, tf, tb, act, st, vs)
    assert mb_off.tolist() == mbo
    host = planner.select_recomputation(shapes, np.array(mbo), W.grid(), model, (0, 1, 2), lim)
    assert st.cpu().numpy().tolist() == host["strategy"].tolist()
    assert vs.cpu().numpy().tolist() == host["violating_stage"].tolist()
    assert len(set(host["strategy"].tolist())) > 1  # the limits really split the strategies
    n = len(shapes)
    for q in range(M):
        if host["strategy"][q] < 0:
            continue
        a, b = mbo[q] * C_, mbo[q + 1] * C_
        for k, d in (("t_f", tf), ("t_b", tb), ("act_mem", act)):
            assert host[k].reshape(-1)[a:b].tobytes() == d[a:b].cpu().numpy().tobytes(), (k, q)
    if reference_available():
        exp = Reference().select_recomputation(shapes, np.array(mbo), W.grid(), model, (0, 1, 2), lim)
        assert exp["strategy"].tolist() == host["strategy"].tolist()


def test_pack_plan_slots_kernel_matches_host_packing(planner):
    """pp_pack_plan_slots (csrc/slots.cu) packs device plans into exactly the
    slots shard.pack_slots builds on the host, order included; unpacked
    slots give the reference's MicroBatch sample_ids."""
    import torch

    from paper_2311_10418_b200 import shard

    cfg = W.CONFIGS["C1"]
    M, n = 7, cfg.n
    s = W.dataset(cfg, M)
    s[:, 0] = np.random.default_rng(5).permutation(len(s)) + 100  # ids unrelated to positions
    off = W.seg_offsets(cfg, M)
    d_s = torch.from_numpy(s).cuda()
    out = {"ordered": torch.empty((M * n, 3), dtype=torch.int64, device="cuda"),
           "order": torch.empty(M * n, dtype=torch.int32, device="cuda"),
           "splits": torch.empty(M * n, dtype=torch.int32, device="cuda"),
           "mb_times": torch.empty(M * n, dtype=torch.float64, device="cuda"),
           "count": torch.empty(M, dtype=torch.int32, device="cuda"),
           "t_max_used": torch.empty(M, dtype=torch.float64, device="cuda"),
           "objective": torch.empty(M, dtype=torch.float64, device="cuda"),
           "status": torch.empty(M, dtype=torch.int32, device="cuda"),
           "err_sample_id": torch.empty(M, dtype=torch.int64, device="cuda")}
    slots = shard.plan_shard_device(planner, d_s, n, M, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap,
                                    cfg.interval, out)
    torch.cuda.synchronize()
    host = shard.pack_slots(out["count"].cpu(), out["status"].cpu(), out["t_max_used"].cpu(),
                            out["objective"].cpu(), out["splits"].cpu(), n, out["order"].cpu())
    assert torch.equal(slots.cpu(), host)
    orc = Oracle()
    for k, plan in enumerate(shard.unpack_slots(slots, n)):
        mb = s[off[k]:off[k + 1]]
        ref = orc.plan(mb, W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
        assert np.array_equal(plan["splits"], ref.splits)
        lo = 0
        for e, ids in zip(ref.splits, shard.micro_batch_sample_ids(mb, plan)):
            assert np.array_equal(ids, ref.ordered[lo:e, 0])
            lo = e
