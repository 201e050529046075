"""Seeded op-cost tables for the injection-order search:
order_microbatches + the planner's simulate(plan_communication(...)) evaluator
(proj/src/schedule.cpp:277-317, planner.cpp:94-108).

Each case is (name, t_f, t_b, act, mb_offset, limits, n_clusters,
comm_latency) with tables shaped (rows, stages) like OpCostTable
(cost_model.h:148-171).  Durations are drawn on a coarse lattice so equal
makespans (the identity tie rule, schedule.cpp:307-312) and equal transfer
ends (the (end, device, op_index) sort, comm_plan.cpp:150-152) occur."""
from __future__ import annotations

import numpy as np


def random_tables(rng, n_tab, m_lo, m_hi, C, lattice=True, act_scale=1.0):
    ms = rng.integers(m_lo, m_hi + 1, size=n_tab)
    off = np.concatenate([[0], np.cumsum(ms)]).astype(np.int64)
    rows = int(off[-1])
    if lattice:
        tf = rng.integers(1, 9, size=(rows, C)).astype(np.float64) * 0.25
        tb = rng.integers(1, 9, size=(rows, C)).astype(np.float64) * 0.5
    else:
        tf = rng.lognormal(0.0, 0.6, size=(rows, C))
        tb = 2.0 * tf * rng.uniform(0.9, 1.1, size=(rows, C))
    act = rng.uniform(0.1, 1.0, size=(rows, C)) * act_scale
    return tf, tb, act, off


def cases(seed=2311, big=False):
    rng = np.random.default_rng(seed)
    out = []
    # (M range, stages, clusters, limit factor over max act, latency, lattice)
    grid = [
        ((1, 1), 1, 3, 4.0, 0.0, True),
        ((1, 3), 4, 3, 4.0, 0.0, True),
        ((2, 6), 2, 3, 3.0, 0.0, True),
        ((4, 12), 4, 3, 2.5, 0.0, True),
        ((8, 24), 4, 1, 4.0, 0.0, True),
        ((8, 24), 8, 2, 3.0, 0.25, True),
        ((10, 40), 4, 4, 1.6, 0.0, True),
        ((10, 40), 5, 5, 6.0, 0.5, False),
        ((16, 48), 16, 3, 2.0, 0.0, True),
        ((20, 60), 3, 3, 1e300, 0.0, False),
        ((6, 20), 32, 3, 3.0, 0.125, True),
        ((30, 80), 8, 3, 2.0, 1.0, False),
    ]
    if big:
        grid += [((150, 400), 4, 3, 3.0, 0.0, False), ((200, 600), 8, 4, 2.0, 0.25, True),
                 ((400, 900), 16, 3, 4.0, 0.0, False)]
    for q, ((lo, hi), C, k, fac, lat, lattice) in enumerate(grid):
        tf, tb, act, off = random_tables(rng, 6 if not big or q < len(grid) - 3 else 3, lo, hi, C, lattice)
        lim = fac * act.max(axis=0) if fac < 1e300 else np.full(C, 1e300)
        out.append((f"rand{q}_C{C}_k{k}", tf, tb, act, off, lim, k, lat))
    # uniform costs: every order ties, the identity order must win
    C, M = 4, 12
    tf = np.full((M, C), 1.0)
    out.append(("uniform", tf, 2.0 * tf, np.full((M, C), 0.5), np.array([0, M], np.int64), np.full(C, 3.0), 3,
                0.0))
    # two-valued costs: clusters of equal predicted time
    rows = 30
    tf = np.where(np.arange(rows)[:, None] % 3 == 0, 2.0, 1.0) * np.ones((rows, 4))
    out.append(("twovalued", tf, tf * 2, np.full((rows, 4), 0.3), np.array([0, 10, 30], np.int64),
                np.full(4, 1.0), 3, 0.0))
    return out


def nonconvergent():
    """One act above its device limit: the forward can never be admitted
    (schedule.cpp:80-82 throws logic_error)."""
    tf = np.ones((5, 3))
    act = np.full((5, 3), 0.5)
    act[2, 1] = 5.0
    return tf, tf * 2, act, np.array([0, 5], np.int64), np.full(3, 2.0)
