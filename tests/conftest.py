import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def load_golden(name):
    path = os.path.join(GOLDEN, name + ".json")
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name}.json not generated")
    with open(path) as f:
        return json.load(f)


def toy_tables(lens, mem_per_sample=0.0, heavy=False):
    """proj/tests/test_microbatch.cpp:37-46 toy coster as triangular tables:
    t(M) = max_len * |M|, mem = k * |M| (heavy: mem = t)."""
    import numpy as np
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


def record(p, with_order=True):
    """A checker plan as a golden-style record."""
    rec = dict(status=int(p.status), err_sample_id=int(p.err_sample_id))
    if p.status == 0:
        rec.update(splits=[int(x) for x in p.splits], mb_times=[float(x).hex() for x in p.mb_times],
                   t_max_used=float(p.t_max_used).hex(), objective=float(p.objective).hex())
        if with_order and getattr(p, "ordered", None) is not None:
            rec["ordered_ids"] = [int(x) for x in p.ordered[:, 0]]
        if getattr(p, "replica", None) is not None:
            rec["replica"] = [int(x) for x in p.replica]
            rec["max_load"] = float(p.max_load).hex()
    if getattr(p, "n_candidates", -1) >= 0:
        rec["n_candidates"] = int(p.n_candidates)
        rec["n_evaluated"] = int(p.n_evaluated)
    return rec


def unhex(x):
    return float.fromhex(x) if isinstance(x, str) else float(x)


def assert_plan_matches(got, expect, ctx=""):
    """Bit-exact parity with a golden/checker record: status
    and error sample, splits, slice times, t_max_used, objective (1e-6), the
    ordering, dp_partition's replica assignment and max_replica_load, and the
    candidate loop's counters (|candidates|, candidates the reference's loop
    visits) whenever both sides carry them."""
    assert int(got.status) == expect["status"], f"{ctx}: status {got.status} != {expect['status']}"
    if "n_candidates" in expect and getattr(got, "n_candidates", -1) >= 0 and expect["status"] == 0:
        assert int(got.n_candidates) == expect["n_candidates"], \
            f"{ctx}: candidates {got.n_candidates} != {expect['n_candidates']}"
        assert int(got.n_evaluated) == expect["n_evaluated"], \
            f"{ctx}: reference-loop evaluations {got.n_evaluated} != {expect['n_evaluated']}"
    if expect["status"] != 0:
        if expect["status"] == 2:
            assert int(got.err_sample_id) == expect["err_sample_id"], ctx
        return
    assert [int(x) for x in got.splits] == expect["splits"], f"{ctx}: splits differ"
    assert [float(x).hex() for x in got.mb_times] == expect["mb_times"], f"{ctx}: times differ"
    assert float(got.t_max_used).hex() == expect["t_max_used"], f"{ctx}: t_max_used differs"
    obj, eobj = float(got.objective), unhex(expect["objective"])
    assert obj == eobj or abs(obj - eobj) <= 1e-6 * abs(eobj), f"{ctx}: objective {obj} != {eobj}"
    if "ordered_ids" in expect and getattr(got, "ordered", None) is not None:
        assert [int(x) for x in got.ordered[:, 0]] == expect["ordered_ids"], f"{ctx}: order differs"
    if "replica" in expect and getattr(got, "replica", None) is not None:
        assert [int(x) for x in got.replica] == expect["replica"], f"{ctx}: replica assignment differs"
        assert float(got.max_load).hex() == expect["max_load"], f"{ctx}: max_replica_load differs"
