"""CPU: the C-ABI library loads, exports every symbol include/pipeplan_b200.h
declares, refuses to plan without a device (no CPU fallback), and its
host-side helpers reproduce the reference bit-for-bit."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from oracle.bind import Oracle, Reference, reference_available
from paper_2311_10418_b200 import capi
from paper_2311_10418_b200 import workloads as W

HEADER = os.path.join(ROOT, "include", "pipeplan_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(pp_\w+)\s*\(", text, re.M)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(capi.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(capi._LIB_PATH)
    for sym in declared_symbols():
        assert hasattr(lib, sym), sym
    assert lib.pp_abi_version() == 1


def test_library_has_sm100a_code():
    data = open(capi._LIB_PATH, "rb").read()
    assert b"sm_100a" in data


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES") != "" and __import__("torch").cuda.is_available(),
                    reason="a device is present")
def test_no_device_means_no_planner():
    with pytest.raises(capi.NoDeviceError):
        capi.Planner()


def test_synthetic_grid_matches_reference_defaults():
    g = capi.synthetic_grid()
    assert list(g.mbs_axis) == [1 << k for k in range(9)]
    assert list(g.seq_axis) == [32 << k for k in range(12)]
    if reference_available():
        mb, sq, cells = Reference().synthetic_grid_cells(
            [0.4, 2e-4, 0.02, 0.2, 0.6, 1.0, 0.5], 1)
        assert np.array_equal(mb, g.mbs_axis) and np.array_equal(sq, g.seq_axis)
        assert cells.tobytes() == g.cells.tobytes()


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
def test_synthetic_dataset_is_byte_identical_to_reference():
    ref = Reference()
    for n, L, seed, tgt in [(1000, 8192, 7, None), (777, 65536, 3, W.T5_TARGET_DIST),
                            (500, 300, 11, (capi.MIXTURE, 4.0, 1.0, 5, 900, 0.7)),
                            (300, 100, 1, (capi.UNIFORM, 0, 0, 1, 50, 0))]:
        a = capi.synthetic_dataset(n, L, seed, W.INPUT_DIST, tgt)
        b = ref.load_dataset(n, L, seed, W.INPUT_DIST, tgt)
        assert a.tobytes() == b.tobytes()


def test_dataset_statistics_match_survey():
    s = W.dataset(W.CONFIGS["C3"], 1)
    x = s[:, 1]
    assert np.median(x) == pytest.approx(147, abs=8)  # p50 147
    assert x.max() == 8192


def test_host_slice_cost_matches_oracle():
    orc = Oracle()
    grid = W.grid()
    rng = np.random.default_rng(1)
    for encdec in (False, True):
        model = capi.Model.uniform(6, 2, encdec)
        s = capi.synthetic_dataset(300, 8192, 9, W.INPUT_DIST, W.T5_TARGET_DIST if encdec else None)
        for _ in range(50):
            b = int(rng.integers(0, 299))
            e = int(rng.integers(b + 1, 301))
            assert capi.slice_cost_host(grid, model, s, b, e) == orc.slice_cost(grid, model, s, b, e)


def test_eval_objective_closed_form():
    # proj/tests/test_microbatch.cpp:132-137
    assert capi.eval_objective([4, 6, 10], 4, 1) == 50
    assert capi.eval_objective([4, 6, 10], 1, 1) == 20
    assert capi.eval_objective([4, 6, 10], 4, 2) == 40
    with pytest.raises(capi.InvalidArgument):
        capi.eval_objective([], 1, 1)


def test_frozen_intervals_rederive():
    """workloads.py's frozen I (mapping A') re-derived with the oracle."""
    orc = Oracle()
    for name in ("C1", "C2"):
        cfg = W.CONFIGS[name]
        o = orc.order_samples(W.dataset(cfg, 1))
        tcap, _ = orc.slice_extrema(o, W.grid(), W.model(cfg), cfg.mem_cap)
        assert tcap / cfg.K == cfg.interval


def test_model_uniform_layouts():
    m = capi.Model.uniform(8, 2, True)
    assert list(m.encoder_layers) == [2, 2, 2, 2, 0, 0, 0, 0]
    assert list(m.decoder_layers) == [0, 0, 0, 0, 2, 2, 2, 2]
    m = capi.Model.uniform(5, 3, True)
    assert list(m.encoder_layers) == [3, 3, 3, 0, 0]
    m = capi.Model.uniform(1, 2, True)
    assert list(m.encoder_layers) == [2] and list(m.decoder_layers) == [2]
    m = capi.Model.uniform(4, 2, False)
    assert list(m.encoder_layers) == [0] * 4 and list(m.decoder_layers) == [2] * 4
