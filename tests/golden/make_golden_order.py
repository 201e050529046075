"""Golden fixtures for the injection-order search,
generated from the UNMODIFIED reference (oracle/_ref: proj/src/schedule.cpp,
comm_plan.cpp, simulate.cpp compiled where they lie):

    python tests/golden/make_golden_order.py   ->  tests/golden/order_search.json

Inputs are the seeded tables of tests/order_cases.py (stored too, as hex, so
the fixture does not depend on numpy's generator); expected outputs are the
reference's order_microbatches result with plan_iteration's evaluator and the
chosen order's SimReport (planner.cpp:94-108), doubles as float.hex()."""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle.bind import Reference, build  # noqa: E402
from order_cases import cases, nonconvergent  # noqa: E402


def hx(a):
    return [float(x).hex() for x in np.asarray(a, np.float64).ravel()]


def main():
    build(ref=True)
    R = Reference()
    out = []
    todo = list(cases()) + [("nonconvergent",) + nonconvergent()[:4] + (nonconvergent()[4], 3, 0.0)]
    for name, tf, tb, act, off, lim, k, lat in todo:
        _, o = R.order_search(tf, tb, act, off, lim, k, lat)
        out.append(dict(name=name, stages=int(tf.shape[1]), n_clusters=int(k), comm_latency=float(lat).hex(),
                        t_f=hx(tf), t_b=hx(tb), act=hx(act), mb_offset=[int(x) for x in off], limits=hx(lim),
                        expect=dict(status=[int(x) for x in o["status"]], order=[int(x) for x in o["order"]],
                                    makespan=hx(o["makespan"]), bubble_ratio=hx(o["bubble_ratio"]),
                                    deadlock=[int(x) for x in o["deadlock"]],
                                    device_stats=hx(o["device_stats"]))))
    with open(os.path.join(HERE, "order_search.json"), "w") as f:
        json.dump(out, f)
    print(f"{len(out)} cases -> order_search.json")


if __name__ == "__main__":
    main()
