"""Whole-epoch planning across GPUs: shard mini-batches, plan locally, gather plans.

The reference plans independent mini-batches on run_plan's std::thread pool
(src/driver.cpp:222-242) and keeps every MicroBatchPartition.  Here each rank
(one process per GPU) plans a contiguous block of mini-batches through the
C-ABI, ONE kernel (pp_pack_plan_slots) packs the plans into fixed-size slots,
and ONE all_gather of the slots makes the whole epoch's plans visible on every
rank.  There is no other collective: planning itself never communicates.

Slot layout (int64 words, one slot per mini-batch; csrc/slots.cu):
    [0] micro-batch count   [1] status   [2] t_max_used (float64 bits)
    [3] objective (float64 bits)   [4 : 4 + h] splits as packed int32
    [4 + h : 4 + 2h] (with_order) the ordering as packed int32 per-segment
                     sample indices, h = ceil(n / 2)
Micro-batch k of a plan holds the samples order[splits[k-1] : splits[k]] of
its mini-batch: that is make_micro_batch's sample_ids (microbatch.cpp:122-134)
once the ids of the mini-batch's input samples are looked up.
The backend is whatever the process group uses (NCCL on the B200 box, gloo in
the CPU tests).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

HEADER_WORDS = 4
PAD_STATUS = -1  # status of the padding slots of a short shard (never a plan)


def shard_range(n_minibatches: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced block [lo, hi) of mini-batches for `rank`
    (equal-size mini-batches cost the same)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, extra = divmod(n_minibatches, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def slot_words(n: int, with_order: bool = True) -> int:
    return HEADER_WORDS + (2 if with_order else 1) * ((n + 1) // 2)


def pack_slots(count, status, t_max_used, objective, splits, n: int, order=None) -> torch.Tensor:
    """Plans of M mini-batches of n samples each -> (M, slot_words(n)) int64,
    with framework ops (the host-side form of pp_pack_plan_slots, used by the
    CPU tests; the device path packs with Planner.pack_slots_device)."""
    count = torch.as_tensor(count)
    M = count.shape[0]
    dev = count.device
    with_order = order is not None
    h = (n + 1) // 2
    slot = torch.zeros((M, slot_words(n, with_order)), dtype=torch.int64, device=dev)
    st = torch.as_tensor(status, device=dev).to(torch.int64)
    ok = st == 0
    slot[:, 0] = torch.where(ok, count.to(torch.int64), torch.zeros_like(st))
    slot[:, 1] = st
    slot[:, 2] = torch.as_tensor(t_max_used, dtype=torch.float64, device=dev).view(torch.int64) * ok
    slot[:, 3] = torch.as_tensor(objective, dtype=torch.float64, device=dev).view(torch.int64) * ok

    def packed(a):
        a = torch.as_tensor(a, dtype=torch.int32, device=dev).reshape(M, n)
        if n % 2:
            a = torch.cat([a, torch.zeros((M, 1), dtype=torch.int32, device=dev)], 1)
        return a.contiguous().view(torch.int64).view(M, -1)

    sp = torch.as_tensor(splits, dtype=torch.int32, device=dev).reshape(M, n).clone()
    sp[torch.arange(n, device=dev)[None, :] >= slot[:, 0:1]] = 0
    slot[:, HEADER_WORDS:HEADER_WORDS + h] = packed(sp)
    if with_order:
        slot[:, HEADER_WORDS + h:] = packed(order)
    return slot


def unpack_slots(slots: torch.Tensor, n: int, with_order: bool = True) -> list[dict]:
    """Inverse of pack_slots / pp_pack_plan_slots for a (..., slot_words(n)) tensor."""
    s = slots.reshape(-1, slot_words(n, with_order)).cpu()
    h = (n + 1) // 2
    out = []
    for row in s:
        m = int(row[0])
        sp = row[HEADER_WORDS:HEADER_WORDS + h].clone().view(torch.int32)[:n]
        rec = {"count": m, "status": int(row[1]),
               "t_max_used": float(row[2:3].view(torch.float64)[0]),
               "objective": float(row[3:4].view(torch.float64)[0]),
               "splits": sp[:m].numpy().astype(np.int32)}
        if with_order:
            rec["order"] = row[HEADER_WORDS + h:].clone().view(torch.int32)[:n].numpy().astype(np.int32)
        out.append(rec)
    return out


def micro_batch_sample_ids(samples: np.ndarray, plan: dict) -> list[np.ndarray]:
    """make_micro_batch's sample_ids (microbatch.cpp:122-134) of one gathered
    plan, from its mini-batch's input samples ((n, 3): id, input, target)."""
    ids = np.asarray(samples)[:, 0][plan["order"]]
    out, lo = [], 0
    for e in plan["splits"]:
        out.append(ids[lo:int(e)])
        lo = int(e)
    return out


def gather_epoch(local_slots: torch.Tensor, n_minibatches: int, group=None) -> torch.Tensor:
    """all_gather of the ranks' slot blocks -> (n_minibatches, words), every
    rank.  Shards from shard_range may differ in size by one: each block is
    padded to ceil(M / world) slots with PAD_STATUS before the collective
    (all_gather_into_tensor needs equal sizes on every rank) and the padding
    is dropped after it, so any M works."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_range(n_minibatches, world, rank)
    if local_slots.shape[0] != hi - lo:
        raise ValueError(f"rank {rank} holds {local_slots.shape[0]} slots, shard_range says {hi - lo}")
    if world == 1:
        return local_slots
    per = -(-n_minibatches // world)
    words = local_slots.shape[1]
    blk = local_slots
    if blk.shape[0] < per:
        pad = torch.zeros((per - blk.shape[0], words), dtype=blk.dtype, device=blk.device)
        pad[:, 1] = PAD_STATUS
        blk = torch.cat([blk, pad], 0)
    out = torch.empty((world * per, words), dtype=blk.dtype, device=blk.device)
    dist.all_gather_into_tensor(out, blk.contiguous(), group=group)
    if n_minibatches % world == 0:
        return out
    keep = torch.cat([torch.arange(r * per, r * per + (b - a), device=out.device)
                      for r, (a, b) in ((r, shard_range(n_minibatches, world, r)) for r in range(world))])
    return out.index_select(0, keep)


def gather_plans(slot: torch.Tensor, group=None) -> torch.Tensor:
    """all_gather of EQUAL-size local slot blocks -> (world * M, words); for
    shards of unequal size use gather_epoch."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return slot
    n_local = torch.tensor([slot.shape[0]], device=slot.device)
    sizes = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(sizes, n_local, group=group)
    if any(int(x) != slot.shape[0] for x in sizes):
        raise ValueError("gather_plans needs equal slot counts on every rank (use gather_epoch)")
    out = torch.empty((world * slot.shape[0], slot.shape[1]), dtype=slot.dtype, device=slot.device)
    dist.all_gather_into_tensor(out, slot.contiguous(), group=group)
    return out


def plan_shard_device(planner, d_samples, n: int, M: int, grid, model, stage_count: int,
                      replica_count: int, mem_cap: float, interval: float, out: dict,
                      d_seg=None, seg=None, slots=None, with_order: bool = True) -> torch.Tensor:
    """Plan M resident mini-batches of n samples (device tensors) and return
    their packed slots on the device (written into `slots` when given).
    `out` needs the pp_plan_out fields, 'order' among them when with_order."""
    if seg is None:
        seg = np.arange(M + 1, dtype=np.int64) * n
    if d_seg is None:
        d_seg = torch.from_numpy(seg).to(d_samples.device)
    planner.plan_batch_device(d_samples, d_seg, seg, out, grid, model, stage_count, replica_count,
                              mem_cap, interval)
    if slots is None:
        slots = torch.empty((M, slot_words(n, with_order)), dtype=torch.int64, device=d_samples.device)
    planner.pack_slots_device(out, d_seg, M, n, slots, with_order)
    return slots
