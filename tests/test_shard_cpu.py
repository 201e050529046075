"""CPU: the multi-GPU sharding / plan-gather host logic with world_size 2 over
gloo.  Each rank plans its shard of mini-batches (with the C restatement as a
stand-in for the device planner — test-only), packs the plans into slots and
all_gathers them; every rank must then hold the whole epoch's plans in order,
bit-exact."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.bind import Oracle
from paper_2311_10418_b200 import capi, shard
from paper_2311_10418_b200 import workloads as W


def test_shard_range_covers_everything():
    for total in (0, 1, 7, 4096):
        for world in (1, 2, 3, 8):
            got = [shard.shard_range(total, world, r) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            sizes = [hi - lo for lo, hi in got]
            assert max(sizes) - min(sizes) <= 1


def test_pack_roundtrip_odd_and_even():
    rng = np.random.default_rng(0)
    for n in (1, 2, 7, 64):
        M = 3
        count = rng.integers(1, n + 1, M).astype(np.int32)
        splits = np.zeros((M, n), np.int32)
        for k in range(M):
            splits[k, :count[k]] = np.sort(rng.choice(np.arange(1, n + 1), count[k], replace=False))
            splits[k, count[k] - 1] = n
        tm = rng.random(M) * 1e6
        ob = rng.random(M) * 1e7
        st = np.zeros(M, np.int32)
        slots = shard.pack_slots(torch.from_numpy(count), torch.from_numpy(st), torch.from_numpy(tm),
                                 torch.from_numpy(ob), torch.from_numpy(splits), n)
        back = shard.unpack_slots(slots, n, False)
        for k in range(M):
            assert back[k]["count"] == count[k]
            assert back[k]["t_max_used"] == tm[k] and back[k]["objective"] == ob[k]
            assert np.array_equal(back[k]["splits"], splits[k, :count[k]])
        order = np.stack([rng.permutation(n) for _ in range(M)]).astype(np.int32)
        slots = shard.pack_slots(torch.from_numpy(count), torch.from_numpy(st), torch.from_numpy(tm),
                                 torch.from_numpy(ob), torch.from_numpy(splits), n, torch.from_numpy(order))
        assert slots.shape[1] == shard.slot_words(n, True)
        back = shard.unpack_slots(slots, n, True)
        for k in range(M):
            assert np.array_equal(back[k]["order"], order[k])
            assert np.array_equal(back[k]["splits"], splits[k, :count[k]])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _order_of(samples, ordered):
    """Per-segment sample index of each ordered position (pp_plan_out.order)."""
    pos = {int(i): k for k, i in enumerate(samples[:, 0])}
    return np.array([pos[int(i)] for i in ordered[:, 0]], np.int32)


def _worker(rank, world, port, M, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = W.CONFIGS["C1"]
        data = capi.synthetic_dataset(n * M, 8192, 7, W.INPUT_DIST)
        lo, hi = shard.shard_range(M, world, rank)
        orc = Oracle()
        k_loc = hi - lo
        count = np.zeros(k_loc, np.int32)
        status = np.full(k_loc, -1, np.int32)
        tm = np.zeros(k_loc)
        ob = np.zeros(k_loc)
        splits = np.zeros((k_loc, n), np.int32)
        order = np.zeros((k_loc, n), np.int32)
        for k, mb in enumerate(range(lo, hi)):
            mbs = data[mb * n:(mb + 1) * n]
            p = orc.plan(mbs, W.grid(), W.model(cfg), cfg.stages, 1, math.inf, cfg.interval)
            count[k] = len(p.splits)
            status[k] = p.status
            tm[k] = p.t_max_used
            ob[k] = p.objective
            splits[k, :count[k]] = p.splits
            order[k] = _order_of(mbs, p.ordered)
        slots = shard.pack_slots(torch.from_numpy(count), torch.from_numpy(status), torch.from_numpy(tm),
                                 torch.from_numpy(ob), torch.from_numpy(splits), n, torch.from_numpy(order))
        # unequal shards (M % world != 0): gather_epoch pads and trims
        plans = shard.unpack_slots(shard.gather_epoch(slots, M), n)
        ok = len(plans) == M
        for mb in range(M):
            mbs = data[mb * n:(mb + 1) * n]
            ref = orc.plan(mbs, W.grid(), W.model(cfg), cfg.stages, 1, math.inf, cfg.interval)
            ok &= plans[mb]["status"] == 0 and np.array_equal(plans[mb]["splits"], ref.splits)
            ok &= plans[mb]["t_max_used"] == ref.t_max_used and plans[mb]["objective"] == ref.objective
            # the reference's MicroBatch::sample_ids (microbatch.cpp:122-134)
            ids = shard.micro_batch_sample_ids(mbs, plans[mb])
            lo_ = 0
            for e, got in zip(ref.splits, ids):
                ok &= np.array_equal(got, ref.ordered[lo_:e, 0])
                lo_ = e
        # gather_plans refuses unequal blocks instead of hanging the collective
        try:
            shard.gather_plans(slots)
            ok &= (M % world == 0)
        except ValueError:
            ok &= (M % world != 0)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_epoch_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    M, n = 5, 96
    procs = [ctx.Process(target=_worker, args=(r, 2, port, M, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
