"""Injection-order search: the device kernels behind
pp_order_search against the UNMODIFIED reference's order_microbatches with
plan_iteration's evaluator (proj/src/schedule.cpp:277-317, comm_plan.cpp:115-233,
simulate.cpp:78-213, planner.cpp:94-108).  Bit-exact: the chosen order, the
makespan / bubble ratio / per-device stats (compared as float bit patterns),
the deadlock flag and the error status."""
import math

import numpy as np
import pytest

from conftest import load_golden
from oracle.bind import Reference, reference_available
from order_cases import cases, nonconvergent, random_tables
from paper_2311_10418_b200 import capi
from paper_2311_10418_b200 import workloads as W


def _unhex(xs, shape=None):
    a = np.array([float.fromhex(x) for x in xs])
    return a.reshape(shape) if shape else a


def _golden_inputs(case):
    C = case["stages"]
    tf = _unhex(case["t_f"], (-1, C))
    return (tf, _unhex(case["t_b"], (-1, C)), _unhex(case["act"], (-1, C)),
            np.array(case["mb_offset"], np.int64), _unhex(case["limits"]), case["n_clusters"],
            float.fromhex(case["comm_latency"]))


def assert_same(got, exp, name):
    st = np.asarray(exp["status"])
    assert np.array_equal(got["status"], st), f"{name}: status {got['status']} != {st}"
    ok = st == 0
    assert np.array_equal(np.asarray(got["order"]), np.asarray(exp["order"])) or not ok.all(), \
        f"{name}: order differs"
    for key in ("makespan", "bubble_ratio"):
        g = np.asarray(got[key], np.float64)[ok]
        e = np.asarray(exp[key], np.float64)[ok]
        assert g.tobytes() == e.tobytes(), f"{name}: {key} {g} != {e}"
    assert np.array_equal(np.asarray(got["deadlock"])[ok], np.asarray(exp["deadlock"])[ok]), name
    g = np.asarray(got["device_stats"], np.float64)[ok]
    e = np.asarray(exp["device_stats"], np.float64).reshape(g.shape[0] if ok.all() else -1, *g.shape[1:])
    if ok.all():
        assert g.tobytes() == e.tobytes(), f"{name}: device stats differ"


# ---- CPU: the fixture is what the reference computes --------------------
@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
def test_golden_matches_live_reference():
    R = Reference()
    for case in load_golden("order_search"):
        tf, tb, act, off, lim, k, lat = _golden_inputs(case)
        _, got = R.order_search(tf, tb, act, off, lim, k, lat)
        exp = dict(case["expect"])
        exp["makespan"] = _unhex(exp["makespan"])
        exp["bubble_ratio"] = _unhex(exp["bubble_ratio"])
        exp["device_stats"] = _unhex(exp["device_stats"], got["device_stats"].shape)
        assert_same(got, exp, case["name"])


def test_golden_cases_regenerate():
    """tests/order_cases.py still generates the stored inputs."""
    golden = {c["name"]: c for c in load_golden("order_search")}
    for name, tf, tb, act, off, lim, k, lat in cases():
        g = golden[name]
        gtf, gtb, gact, goff, glim, gk, glat = _golden_inputs(g)
        assert gtf.tobytes() == tf.tobytes() and gact.tobytes() == act.tobytes(), name
        assert np.array_equal(goff, off) and gk == k and glat == lat, name


# ---- GPU parity ----------------------------------------------------------
@pytest.fixture(scope="module")
def planner():
    p = capi.Planner(0)
    yield p
    p.close()


@pytest.mark.gpu
def test_golden_order_search(planner):
    for case in load_golden("order_search"):
        tf, tb, act, off, lim, k, lat = _golden_inputs(case)
        got = planner.order_search(tf, tb, act, off, lim, k, lat)
        exp = dict(case["expect"])
        exp["makespan"] = _unhex(exp["makespan"])
        exp["bubble_ratio"] = _unhex(exp["bubble_ratio"])
        exp["device_stats"] = _unhex(exp["device_stats"], got["device_stats"].shape)
        assert_same(got, exp, case["name"])


@pytest.mark.gpu
@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
def test_large_random_tables_vs_reference(planner):
    R = Reference()
    for name, tf, tb, act, off, lim, k, lat in cases(seed=77, big=True):
        got = planner.order_search(tf, tb, act, off, lim, k, lat)
        _, exp = R.order_search(tf, tb, act, off, lim, k, lat, threads=8)
        assert_same(got, exp, name)


@pytest.mark.gpu
@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
def test_planner_tables_vs_reference(planner):
    """The planner's own pipeline: device plans (C1-style GPT and a T5
    config) -> device op-cost tables (OpCostTable::from_shapes) -> order
    search; the reference runs order_microbatches on the same tables."""
    import torch
    R = Reference()
    grid = W.grid()
    for encdec, C, n, segs, k in [(False, 4, 256, 12, 3), (True, 8, 512, 4, 3), (False, 16, 1024, 2, 4)]:
        model = capi.Model.uniform(C, 2, encdec)
        s = capi.synthetic_dataset(n * segs, 8192, 11, W.INPUT_DIST, W.T5_TARGET_DIST if encdec else None)
        off = np.arange(segs + 1, dtype=np.int64) * n
        res = planner.plan_batch(s, off, grid, model, C, 1, math.inf, 5000.0)
        shapes = []
        mb_off = [0]
        for q in range(segs):
            ordered = res["ordered"][off[q]:off[q + 1]]
            sp = res["splits"][off[q]:off[q] + res["count"][q]]
            a = 0
            for e in sp:
                blk = ordered[a:e]
                shapes.append((e - a, max(0, blk[:, 1].max()), max(0, blk[:, 2].max())))
                a = e
            mb_off.append(len(shapes))
        tf, tb, act = planner.op_costs(np.array(shapes, np.int64), grid, model)
        lim = np.full(C, 2.5 * act.max())
        got = planner.order_search(tf, tb, act, np.array(mb_off), lim, k, 0.0)
        _, exp = R.order_search(tf, tb, act, np.array(mb_off), lim, k, 0.0, threads=8)
        assert_same(got, exp, f"planner C={C} encdec={encdec}")
        # device-resident entry point on the same tables
        dev = torch.device("cuda:0")
        d = {key: torch.empty(len(v) if key != "device_stats" else v.shape, dtype=torch.int32
                              if v.dtype == np.int32 else torch.float64, device=dev) for key, v in exp.items()}
        planner.order_search_device(*(torch.from_numpy(x).to(dev) for x in (tf, tb, act)),
                                    torch.tensor(mb_off, dtype=torch.int64, device=dev), mb_off, lim, d, k, 0.0)
        assert_same({key: v.cpu().numpy() for key, v in d.items()}, exp, f"device C={C}")


@pytest.mark.gpu
@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("k, n_tab", [(9, 2), (9, 12), (10, 1)])
def test_more_than_eight_clusters_vs_reference(planner, k, n_tab):
    """n_clusters 9 and 10 (9! = 362,880 / 10! = 3,628,800 evaluations per
    table, as the reference's std::next_permutation loop): one launch for 2
    tables, permutation windows folded into a running best for 12 tables
    (> 4 M evaluations) and for 10 clusters; order, makespan, bubble ratio
    and device stats against the reference's order_microbatches."""
    rng = np.random.default_rng(900 + k + n_tab)
    # (distinct durations for 9 clusters: k-means keeps all k clusters, so
    # every table really has 9! permutations; lattice durations for 10)
    tf, tb, act, off = random_tables(rng, n_tab, k + 2, k + 6, 3, lattice=k > 9)
    lim = 3.0 * act.max(axis=0)
    got = planner.order_search(tf, tb, act, off, lim, k, 0.0)
    _, exp = Reference().order_search(tf, tb, act, off, lim, k, 0.0, threads=16)
    assert_same(got, exp, f"k={k} tables={n_tab}")


def _peer(kind, j):
    return j + 1 if kind in (2, 5, 6, 9) else j - 1


@pytest.mark.gpu
@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("one_f_one_b", [False, True])
def test_emit_plans_vs_reference(planner, one_f_one_b):
    """pp_emit_plans: the instruction lists of plan_communication(schedule_
    adaptive(costs, limits, order)) (or of the 1F1B schedule) for the orders
    the device search chose, against the reference's plan_communication on
    the same order — kinds, micro-batches, peers — plus the SimReport
    summary, and save_plan's text (pp_format_plan) for a T5 and a GPT model."""
    R = Reference()
    for name, tf, tb, act, off, lim, k, lat in cases(seed=5150):
        if name == "uniform" or tf.shape[1] > 16:
            continue
        found = planner.order_search(tf, tb, act, off, lim, k, lat)
        order = found["order"]
        ok = found["status"] == 0
        got = planner.emit_plans(tf, tb, act, off, lim, order, lat, one_f_one_b)
        exp = R.emit_plans(tf, tb, act, off, lim, order, lat, one_f_one_b)
        for s in range(len(off) - 1):
            if not one_f_one_b and (not ok[s] or order[off[s]] < 0):
                continue
            assert got["status"][s] == exp["status"][s], (name, s)
            if exp["status"][s] != 0:
                continue
            C_ = tf.shape[1]
            for j in range(C_):
                a, b = got["instructions"][s][j], exp["instructions"][s][j]
                assert a.tobytes() == b.tobytes(), (name, s, j)
                assert [_peer(int(x), j) for x in a[:, 0] if x >= 2] == [int(p) for p, x in
                                                                         zip(exp["peers"][s][j], b[:, 0]) if x >= 2]
            for key in ("makespan", "bubble_ratio", "deadlock"):
                assert got[key][s] == exp[key][s] or (got[key][s] != got[key][s] and exp[key][s] != exp[key][s]), key
            assert got["device_stats"][s].tobytes() == exp["device_stats"][s].tobytes()
            if not one_f_one_b:  # the adaptive plan reproduces the search's report
                assert got["makespan"][s] == found["makespan"][s]
    # plan text: shapes / model metadata from a real planner table
    rng = np.random.default_rng(3)
    for encdec, C_ in ((True, 4), (False, 3)):
        M = 9
        tf, tb, act, off = random_tables(rng, 1, M, M, C_, lattice=False)
        shapes = np.stack([rng.integers(1, 64, M), rng.integers(1, 4096, M),
                           rng.integers(0, 512, M) if encdec else np.zeros(M, np.int64)], 1).astype(np.int64)
        model = capi.Model.uniform(C_, 2, encdec, recompute=int(rng.integers(0, 3)))
        lim = 3.0 * act.max(axis=0)
        order = planner.order_search(tf, tb, act, off, lim, 3, 0.0)["order"]
        got = planner.emit_plans(tf, tb, act, off, lim, order, 0.0, one_f_one_b)
        text = capi.Planner.format_plan(got["instructions"][0], shapes, model, iteration=7, replica=1, hidden_dim=2048)
        exp = R.emit_plans(tf, tb, act, off, lim, order, 0.0, one_f_one_b, shapes=shapes, model=model, iteration=7,
                           replica=1, hidden=2048)
        assert text == exp["plan_text"], (encdec, text[:200], exp["plan_text"][:200])


@pytest.mark.gpu
def test_errors(planner):
    tf, tb, act, off, lim = nonconvergent()
    got = planner.order_search(tf, tb, act, off, lim)
    assert got["status"][0] == capi.PP_ERR_NOT_CONVERGED
    # a table with no micro-batch, next to a valid one
    t = np.ones((3, 2))
    got = planner.order_search(t, t, t * 0.1, np.array([0, 0, 3]), np.full(2, 1.0))
    assert list(got["status"]) == [capi.PP_ERR_INVALID, 0]
    # negative durations are outside the device path's contract
    got = planner.order_search(-t, t, t * 0.1, np.array([0, 3]), np.full(2, 1.0))
    assert got["status"][0] == capi.PP_ERR_INVALID
    with pytest.raises(capi.InvalidArgument):
        planner.order_search(t, t, t, np.array([0, 3]), np.full(2, 1.0), n_clusters=0)
    with pytest.raises(capi.InvalidArgument):
        planner.order_search(np.ones((3, 33)), np.ones((3, 33)), np.ones((3, 33)), np.array([0, 3]),
                             np.ones(33))
