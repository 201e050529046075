"""Probe: planning G groups of M mini-batches on G contexts (streams) from G
host threads, so one group's latency-bound DP overlaps another's cost passes."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_10418_b200 import capi  # noqa: E402
from paper_2311_10418_b200 import workloads as W  # noqa: E402


def run(name, M, G, reps=5):
    cfg = W.CONFIGS[name]
    n = cfg.n
    data = [torch.from_numpy(capi.synthetic_dataset(M * n, cfg.max_seq_len, 7 + g, W.INPUT_DIST,
                                                    W.T5_TARGET_DIST if cfg.encdec else None)).cuda()
            for g in range(G)]
    seg = W.seg_offsets(cfg, M)
    d_seg = torch.from_numpy(seg).cuda()
    planners = [capi.Planner(0) for _ in range(G)]
    streams = [torch.cuda.Stream() for _ in range(G)]
    for p, s in zip(planners, streams):
        p.set_stream(s.cuda_stream)
    tot = M * n
    outs = [{"ordered": torch.empty((tot, 3), dtype=torch.int64, device="cuda"),
             "splits": torch.empty(tot, dtype=torch.int32, device="cuda"),
             "mb_times": torch.empty(tot, dtype=torch.float64, device="cuda"),
             "count": torch.empty(M, dtype=torch.int32, device="cuda"),
             "t_max_used": torch.empty(M, dtype=torch.float64, device="cuda"),
             "objective": torch.empty(M, dtype=torch.float64, device="cuda"),
             "status": torch.empty(M, dtype=torch.int32, device="cuda"),
             "err_sample_id": torch.empty(M, dtype=torch.int64, device="cuda")} for _ in range(G)]
    grid, model = W.grid(), W.model(cfg)

    def work(g):
        planners[g].plan_batch_device(data[g], d_seg, seg, outs[g], grid, model, cfg.stages, 1,
                                      cfg.mem_cap, cfg.interval)

    def once():
        th = [threading.Thread(target=work, args=(g,)) for g in range(G)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        torch.cuda.synchronize()

    once()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        once()
        best = min(best, time.perf_counter() - t0)
    print(f"{name} M={M} x G={G}: {best * 1e3:.2f} ms, {G * M / best:.0f} plans/s", flush=True)


if __name__ == "__main__":
    for spec in sys.argv[1:]:
        name, M, G = spec.split(":")
        run(name, int(M), int(G))
