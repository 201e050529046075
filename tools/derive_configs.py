"""Derive the exact t_max_interval / memory cap of each BASELINE config.

The reference has no "K candidates" knob, only DpOptions::t_max_interval I
(microbatch.h:79-86).  SURVEY.md §8d mapping A': I = T_capmax / K with
T_capmax the largest slice time among memory-feasible slices of the (first)
mini-batch.  C3's cap is 4 x the largest singleton act_mem.

Uses the C restatement (oracle/) — this is benchmark *setup*, run once; the
values are frozen in paper_2311_10418_b200/workloads.py and re-checked by
tests/test_workloads.py.
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle.bind import Oracle  # noqa: E402
from paper_2311_10418_b200 import workloads as W  # noqa: E402


def main(names):
    orc = Oracle()
    for name in names:
        cfg = W.CONFIGS[name]
        samples = W.dataset(cfg, n_minibatches=1)
        grid = W.grid()
        model = W.model(cfg)
        ordered = orc.order_samples(samples)
        _, act1 = orc.slice_extrema(ordered, grid, model, math.inf)
        cap = cfg.cap_mult * act1 if cfg.cap_mult else math.inf
        tcap, _ = orc.slice_extrema(ordered, grid, model, cap)
        interval = tcap / cfg.K
        print(f"{name}: cap={cap!r} ({float(cap).hex()}) T_capmax={tcap!r} "
              f"I={interval!r} ({interval.hex()})", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2", "C3"])
