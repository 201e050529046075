"""padding_vs_packing_report on the device: every row
(padding efficiencies, tokens, simulated time, throughput proxy) bit-exact
against the UNMODIFIED reference (proj/src/simulate.cpp:288-406, oracle/_ref),
over GPT and T5 models, several max_seq_lens, recompute strategies and
iteration caps, including the reference's own test/acceptance settings
(test_simulate.cpp:218-257, acceptance.cpp:368-395)."""
import numpy as np
import pytest

from oracle.bind import Reference, reference_available
from paper_2311_10418_b200 import capi
from paper_2311_10418_b200 import workloads as W

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")]


@pytest.fixture(scope="module")
def planner():
    p = capi.Planner(0)
    yield p
    p.close()


def same(got, exp, name):
    assert got.tobytes() == exp.tobytes(), f"{name}:\n{got}\n!=\n{exp}"


def test_reference_test_settings(planner):
    R = Reference()
    grid = capi.synthetic_grid(mbs_axis=[1, 2, 4, 8, 16, 32, 64], seq_axis=[32, 64, 128, 256])
    s = np.array([[i, 128, 0] for i in range(64)], np.int64)
    m = capi.Model.uniform(2, 1, False)
    same(planner.padding_report(s, [128], grid, m, 1024, 5.0, 3), R.padding_report(s, [128], grid, m, 1024, 5.0, 3)[1],
         "all-equal")
    rng = np.random.default_rng(55)
    s = np.array([[i, int(rng.integers(1024, 2049)) if rng.random() < 0.2 else int(rng.integers(16, 129)), 0]
                  for i in range(200)], np.int64)
    g = W.grid()
    same(planner.padding_report(s, [2048], g, m, 8192, 5.0, 4), R.padding_report(s, [2048], g, m, 8192, 5.0, 4)[1],
         "skewed")


@pytest.mark.parametrize("encdec,C,recompute", [(False, 4, 0), (True, 8, 0), (False, 2, 1), (True, 4, 2)])
def test_synthetic_datasets(planner, encdec, C, recompute):
    R = Reference()
    g = W.grid()
    m = capi.Model.uniform(C, 2, encdec)
    s = capi.synthetic_dataset(6000, 16384, 21 + C, W.INPUT_DIST, W.T5_TARGET_DIST if encdec else None)
    lens = [512, 2048, 8192]
    got = planner.padding_report(s, lens, g, m, 65536, 500.0, 12, recompute)
    _, exp = R.padding_report(s, lens, g, m, 65536, 500.0, 12, recompute)
    same(got, exp, f"C={C} encdec={encdec} r={recompute}")


def test_errors(planner):
    g = W.grid()
    m = capi.Model.uniform(2, 1, False)
    with pytest.raises(capi.InvalidArgument):
        planner.padding_report(np.zeros((0, 3), np.int64), [128], g, m)
    with pytest.raises(capi.InvalidArgument):
        planner.padding_report(np.array([[0, 5, 0]]), [128], g, m, token_budget=0)
