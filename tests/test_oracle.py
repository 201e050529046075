"""CPU: pin the C restatement (oracle/) against the reference's known answers
and the golden fixtures generated from the unmodified reference."""
import math

import numpy as np
import pytest

from conftest import assert_plan_matches, load_golden, record, toy_tables, unhex
from oracle.bind import Oracle, Reference, reference_available
from paper_2311_10418_b200 import capi
from paper_2311_10418_b200 import workloads as W


@pytest.fixture(scope="module")
def orc():
    return Oracle()


def test_known_answers_test_microbatch(orc):
    # proj/tests/test_microbatch.cpp:139-155 worked instance
    T, M = toy_tables([1, 1, 2, 8])
    p = orc.plan_tables(T, M, 4, 2, 1, math.inf, 0.0)
    assert p.objective == 20.0 and list(p.splits) == [2, 3, 4]
    # :157-166 single sample -> c * t
    T, M = toy_tables([7])
    assert orc.plan_tables(T, M, 1, 4, 1, math.inf, 0.0).objective == 28.0
    # :168-178 memory cap
    T, M = toy_tables([4, 4, 4, 4], 1.0)
    p = orc.plan_tables(T, M, 4, 1, 1, 2.0, 0.0)
    assert p.objective == 16.0 and np.all(np.diff(np.concatenate([[0], p.splits])) <= 2)
    # :246-268 infeasible singleton reported by (ordered) index 1
    T, M = toy_tables([2, 9, 3], heavy=True)
    p = orc.plan_tables(T, M, 3, 1, 1, 5.0, 0.0)
    assert p.status == 2 and p.err_sample_id == 1
    # :132-137 eval_objective closed form
    assert orc.eval_objective([4, 6, 10], 4, 1) == 50
    assert orc.eval_objective([4, 6, 10], 1, 1) == 20
    assert orc.eval_objective([4, 6, 10], 4, 2) == 40


def test_known_answers_test_cost_model(orc):
    # proj/tests/test_cost_model.cpp:47-52: 583.68 at (mbs 2, seq 128)
    g = capi.synthetic_grid([1, 2, 4], [32, 64, 128], alpha=1.0, beta=0.01, gamma=0.01)
    assert orc.per_layer(g, 0, 0, 2, 128)[0] == pytest.approx(583.68, rel=1e-12)
    # :55-67 knots exact, midpoints linear
    g = capi.synthetic_grid([1, 2, 4, 8], [32, 64, 128, 256, 512], alpha=0.7, beta=3e-3, gamma=0.01)
    assert orc.per_layer(g, 1, 0, 2, 128)[0] == pytest.approx(0.7 * 2 * 128 + 3e-3 * 2 * 128 * 128,
                                                              rel=1e-12)
    # :94-103 extrapolation beyond the last knot stays non-negative and grows
    a = orc.per_layer(g, 1, 0, 8, 512)[0]
    b = orc.per_layer(g, 1, 0, 16, 1024)[0]
    assert b > a > 0


def test_oracle_matches_golden_toy(orc):
    for case in load_golden("toy"):
        T, M = toy_tables(case["lens"], case["mem_per_sample"], case["heavy"])
        p = orc.plan_tables(T, M, len(case["lens"]), case["stage_count"], case["replica_count"],
                            unhex(case["mem_cap"]), unhex(case["t_max_interval"]))
        assert_plan_matches(p, case["expect"], case["name"])


def test_oracle_matches_golden_grid(orc):
    grid = capi.synthetic_grid()
    for case in load_golden("grid"):
        model = capi.Model.uniform(case["stages"], 2, case["encdec"])
        s = np.array(case["samples"], np.int64)
        p = orc.plan(s, grid, model, case["stages"], case["replica_count"], unhex(case["mem_cap"]),
                     unhex(case["t_max_interval"]))
        assert_plan_matches(p, case["expect"], case["name"])


def test_oracle_matches_golden_c1(orc):
    case = load_golden("c1")
    cfg = W.CONFIGS["C1"]
    p = orc.plan(W.dataset(cfg, 1), W.grid(), W.model(cfg), cfg.stages, 1, cfg.mem_cap, cfg.interval)
    assert_plan_matches(p, case["expect"], "C1")
    assert len(p.splits) == 216  # SURVEY.md §6 (reference: 216 micro-batches)


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
def test_oracle_matches_reference_random(orc):
    ref = Reference()
    grid = capi.synthetic_grid()
    rng = np.random.default_rng(99)
    for k in range(40):
        n = int(rng.integers(1, 90))
        encdec = bool(rng.integers(0, 2))
        C = int(rng.choice([1, 2, 3, 8]))
        s = capi.synthetic_dataset(n, int(rng.choice([512, 8192])), 500 + k, W.INPUT_DIST,
                                   W.T5_TARGET_DIST if encdec else None)
        model = capi.Model.uniform(C, int(rng.integers(1, 4)), encdec, recompute=int(rng.integers(0, 3)))
        interval = float(rng.choice([0.0, 5.0, 250.0, 4000.0]))
        d = int(rng.integers(1, 3))
        a = ref.plan(s, grid, model, C, d, math.inf, interval)
        b = orc.plan(s, grid, model, C, d, math.inf, interval)
        assert_plan_matches(b, record(a), f"random {k}")


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
def test_oracle_sort_matches_reference(orc):
    ref = Reference()
    rng = np.random.default_rng(5)
    for k in range(20):
        n = int(rng.integers(1, 3000))
        s = np.stack([rng.permutation(n) * 7 - 50, rng.integers(-5, 40, n), rng.integers(0, 9, n)], 1)
        assert np.array_equal(orc.order_samples(s), ref.order_samples(s))


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built (needs /root/reference)")
def test_stream_restatement_matches_reference(orc):
    """Pin the STREAMING restatement (oracle/pp_stream.c, which produced
    tests/golden/c5.json) against the unmodified reference for n <= 2048:
    GPT / T5, capped / uncapped, exact and quantised candidate sets (I in {0,
    5, 1e3} plus the BASELINE mapping-A' interval), several stage counts.
    Also against the table restatement's candidate counters."""
    ref = Reference()
    grid = W.grid()
    rng = np.random.default_rng(2311)
    cases = [(2048, False, 16, 4.0, W.CONFIGS["C3"].interval), (2048, True, 8, 0.0, 1e5),
             (1024, True, 8, 0.0, W.CONFIGS["C2"].interval), (1024, False, 4, 2.0, 1e3)]
    for n in (1, 3, 40, 257):
        for encdec in (False, True):
            for cap_mult in (0.0, 3.0):
                for I in (0.0, 5.0, 1e3):
                    cases.append((n, encdec, int(rng.choice([1, 2, 4, 8])), cap_mult, I))
    for n, encdec, C, cap_mult, I in cases:
        s = capi.synthetic_dataset(n, 8192, 900 + n, W.INPUT_DIST, W.T5_TARGET_DIST if encdec else None)
        s[:, 0] = rng.permutation(n) + 10  # the sort has work to do
        model = capi.Model.uniform(C, 2, encdec)
        cap = math.inf
        if cap_mult:
            o = orc.order_samples(s)
            cap = cap_mult * max(orc.slice_cost(grid, model, o, i, i + 1)[1] for i in range(n))
        ctx = f"n{n} {'t5' if encdec else 'gpt'} C{C} cap{cap_mult} I{I}"
        a = orc.plan_stream(s, grid, model, C, 1, cap, I, threads=4)
        b = ref.plan(s, grid, model, C, 1, cap, I)
        assert_plan_matches(a, record(b), ctx)
        if n <= 257:
            t = orc.plan(s, grid, model, C, 1, cap, I)
            assert (a.n_candidates, a.n_evaluated) == (t.n_candidates, t.n_evaluated), ctx


def test_c5_golden_is_the_stream_restatement_output():
    """tests/golden/c5.json carries what its generator recorded; its
    candidate counters are consistent with BASELINE config C5 (256 bins)."""
    g = load_golden("c5")
    e = g["expect"]
    assert e["status"] == 0 and e["count"] == len(e["split_deltas"])
    assert sum(e["split_deltas"]) == W.CONFIGS["C5"].n and min(e["split_deltas"]) >= 1
    assert e["n_candidates"] <= W.CONFIGS["C5"].K + 1 and e["n_evaluated"] >= 1
