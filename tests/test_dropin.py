"""The reference's OWN unit tests for the hot path — proj/tests/test_microbatch.cpp
and test_cost_model.cpp, compiled unmodified against include/pipeplan/ and
linked with libpipeplan_b200.so (tests/cpp/Makefile -> oracle/_ref/dropin_tests).

* GPU: every test case passes on the B200 planner.
* CPU: the cases that plan (dp_partition) fail LOUDLY with the no-device
  error — the library has no CPU fallback — and everything else passes.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_tests")

pytestmark = pytest.mark.skipif(not os.path.exists(BIN), reason="dropin_tests not built (needs /root/reference)")


def _run():
    return subprocess.run([BIN], capture_output=True, text=True, timeout=600)


@pytest.mark.gpu
def test_reference_unit_tests_pass_on_b200():
    r = _run()
    assert r.returncode == 0, r.stdout + r.stderr
    assert "| 0 failed |" in r.stdout, r.stdout


def test_reference_unit_tests_without_device_fail_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a device is present")
    r = _run()
    lines = [ln for ln in r.stderr.splitlines() if "FAILED" in ln]
    assert lines, r.stdout
    assert all("no CUDA device" in ln for ln in lines), r.stderr
    assert "| 17 passed |" in r.stdout, r.stdout  # cost model, ordering helpers, objective, padding


ACC = os.path.join(ROOT, "oracle", "_ref", "acceptance_dropin")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(ACC), reason="acceptance_dropin not built")
def test_reference_acceptance_suite_on_b200(tmp_path):
    """proj/tests/acceptance.cpp (SPEC.md:509-519 criteria) with the
    reference's planner / scheduler / simulator / driver on top of our hot
    path: criterion 1 (200 brute-force DP instances), 7 (padding efficiency),
    8 (packing direction) and 9 (byte-identical run_plan outputs) exercise
    dp_partition through the reference's own callers."""
    r = subprocess.run([ACC], capture_output=True, text=True, timeout=900, cwd=tmp_path)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]


ORD = os.path.join(ROOT, "oracle", "_ref", "order_dropin")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(ORD), reason="order_dropin not built")
def test_injection_order_search_matches_reference_planner(tmp_path):
    """tests/cpp/order_dropin.cpp: pipeplan::b200::search_injection_order(s)
    against the reference's order_microbatches + plan_communication +
    simulate on random tables, and against the injection orders / reports of
    the reference's own plan_iteration."""
    r = subprocess.run([ORD], capture_output=True, text=True, timeout=600, cwd=tmp_path)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    assert "order dropin: OK" in r.stdout, r.stdout


EPO = os.path.join(ROOT, "oracle", "_ref", "epoch_dropin")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(EPO), reason="epoch_dropin not built")
def test_epoch_planning_files_match_reference_run_plan(tmp_path):
    """tests/cpp/epoch_dropin.cpp: pipeplan::b200::plan_epoch (draw, plans,
    select_recomputation, injection-order search, emitted plans — all on the
    device) writes the same plans_index.csv and .plan files, byte for byte,
    as the reference's run_plan (GPT / T5, 1 and 2 replicas, adaptive and
    1F1B policies, restricted strategy sets, limits tight enough to make
    iterations infeasible)."""
    r = subprocess.run([EPO, str(tmp_path)], capture_output=True, text=True, timeout=900, cwd=tmp_path)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    assert r.stdout.strip().endswith("OK"), r.stdout
