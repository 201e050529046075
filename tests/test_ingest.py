"""Dataset ingest on the device: pp_load_records /
pp_draw_minibatches against the UNMODIFIED reference's load_dataset over a
record file (proj/src/workload.cpp:65-127) and run_plan's draw_minibatch
loop (driver.cpp:209-215, workload.cpp:129-146), compiled in oracle/_ref.
Bit-exact: every sample, or the same ParseError (line, byte offset, kind) /
invalid_argument."""
import os

import numpy as np
import pytest

from ingest_cases import EDGE, long_line_case, random_file
from oracle.bind import Reference, reference_available
from paper_2311_10418_b200 import capi

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")]


@pytest.fixture(scope="module")
def planner():
    p = capi.Planner(0)
    yield p
    p.close()


def ref_load(tmp_path, name, data, max_seq_len):
    path = tmp_path / (name + ".tsv")
    path.write_bytes(data)
    return Reference().load_record_file(str(path), max_seq_len, cap=len(data) + 1)


def ours(planner, data, max_seq_len):
    try:
        return capi.PP_OK, planner.load_records(data, max_seq_len), -1, 0, -1
    except capi.ParseError as e:
        return capi.PP_ERR_PARSE, None, e.line, e.byte_offset, e.kind
    except capi.InvalidArgument:
        return capi.PP_ERR_INVALID, None, -1, 0, -1


def check(got, exp, name):
    assert got[0] == exp[0], f"{name}: status {got[0]} != {exp[0]}"
    if exp[0] == capi.PP_OK:
        assert np.array_equal(got[1], exp[1]), f"{name}: samples differ"
    elif exp[0] == capi.PP_ERR_PARSE:
        assert got[2:] == exp[2:], f"{name}: error {got[2:]} != {exp[2:]}"


@pytest.mark.parametrize("name", sorted(EDGE))
def test_edge_files(planner, tmp_path, name):
    for max_len in (8192, 3):
        check(ours(planner, EDGE[name], max_len), ref_load(tmp_path, name, EDGE[name], max_len), name)


def test_long_line_and_large_files(planner, tmp_path):
    cases = {"long_line": long_line_case(), "random_200k": random_file(200_000),
             "random_clean_1m": random_file(1_000_000, seed=9, noise=False)}
    for name, data in cases.items():
        check(ours(planner, data, 8192), ref_load(tmp_path, name, data, 8192), name)
    bad = bytearray(cases["random_200k"])
    bad[len(bad) * 3 // 4] = ord("x")  # a late malformed record
    check(ours(planner, bytes(bad), 8192), ref_load(tmp_path, "bad", bytes(bad), 8192), "late error")


def test_device_entry_point(planner):
    import torch
    data = random_file(50_000, seed=3)
    host = planner.load_records(data, 8192)
    d_bytes = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
    d_out = torch.empty((len(host) + 10, 3), dtype=torch.int64, device="cuda")
    n = planner.load_records_device(d_bytes, len(data), 8192, d_out)
    assert n == len(host) and np.array_equal(d_out[:n].cpu().numpy(), host)


def test_draw_minibatches(planner):
    R = Reference()
    s = planner.load_records(random_file(300_000, seed=11), 8192)
    for budget in (1, 64, 4096, 65536, 1 << 20, 1 << 40, int(s[:, 1:].sum())):
        got = planner.draw_minibatches(s, budget)
        rc, exp = R.draw_all(s, budget)
        assert rc == 0 and np.array_equal(got, exp), f"budget {budget}"
    with pytest.raises(capi.InvalidArgument):
        planner.draw_minibatches(s, 0)
    assert list(planner.draw_minibatches(s[:0], 10)) == [0]
