"""Whole-epoch planning across GPUs: shard mini-batches, plan locally, gather plans.

The reference plans independent mini-batches on run_plan's std::thread pool
(src/driver.cpp:222-242); here each rank (one process per GPU) plans a
contiguous block of mini-batches through the C-ABI and ONE all_gather of
fixed-size plan slots makes the whole epoch's plans visible on every rank.
There is no other collective: planning itself never communicates.

Slot layout (int64 words, one slot per mini-batch):
    [0] micro-batch count   [1] status   [2] t_max_used (float64 bits)
    [3] objective (float64 bits)   [4 : 4 + ceil(n/2)] splits as packed int32
The backend is whatever the process group uses (NCCL on the B200 box, gloo in
the CPU tests).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

HEADER_WORDS = 4


def shard_range(n_minibatches: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced block [lo, hi) of mini-batches for `rank`
    (equal-size mini-batches cost the same)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, extra = divmod(n_minibatches, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def slot_words(n: int) -> int:
    return HEADER_WORDS + (n + 1) // 2


def pack_slots(count, status, t_max_used, objective, splits, n: int) -> torch.Tensor:
    """Plans of M mini-batches of n samples each -> (M, slot_words(n)) int64.
    Works on CPU or CUDA tensors (no host round trip on the device path)."""
    count = torch.as_tensor(count)
    M = count.shape[0]
    dev = count.device
    slot = torch.zeros((M, slot_words(n)), dtype=torch.int64, device=dev)
    slot[:, 0] = count.to(torch.int64)
    slot[:, 1] = torch.as_tensor(status, device=dev).to(torch.int64)
    slot[:, 2] = torch.as_tensor(t_max_used, dtype=torch.float64, device=dev).view(torch.int64)
    slot[:, 3] = torch.as_tensor(objective, dtype=torch.float64, device=dev).view(torch.int64)
    sp = torch.as_tensor(splits, dtype=torch.int32, device=dev).reshape(M, n)
    if n % 2:
        sp = torch.cat([sp, torch.zeros((M, 1), dtype=torch.int32, device=dev)], 1)
    slot[:, HEADER_WORDS:] = sp.contiguous().view(torch.int64).view(M, -1)
    return slot


def unpack_slots(slots: torch.Tensor, n: int) -> list[dict]:
    """Inverse of pack_slots for a (..., slot_words(n)) tensor."""
    s = slots.reshape(-1, slot_words(n)).cpu()
    out = []
    for row in s:
        m = int(row[0])
        sp = row[HEADER_WORDS:].clone().view(torch.int32)[:n]
        out.append({"count": m, "status": int(row[1]),
                    "t_max_used": float(row[2:3].view(torch.float64)[0]),
                    "objective": float(row[3:4].view(torch.float64)[0]),
                    "splits": sp[:m].numpy().astype(np.int32)})
    return out


def gather_plans(slot: torch.Tensor, group=None) -> torch.Tensor:
    """all_gather of equal-size local slot blocks -> (world * M, words)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return slot
    out = torch.empty((world * slot.shape[0], slot.shape[1]), dtype=slot.dtype, device=slot.device)
    dist.all_gather_into_tensor(out, slot.contiguous(), group=group)
    return out


def plan_shard_device(planner, d_samples, n: int, M: int, grid, model, stage_count: int,
                      replica_count: int, mem_cap: float, interval: float, out: dict,
                      d_seg=None, seg=None) -> torch.Tensor:
    """Plan M resident mini-batches of n samples (device tensors) and return
    their packed slots on the device."""
    if seg is None:
        seg = np.arange(M + 1, dtype=np.int64) * n
    if d_seg is None:
        d_seg = torch.from_numpy(seg).to(d_samples.device)
    planner.plan_batch_device(d_samples, d_seg, seg, out, grid, model, stage_count, replica_count,
                              mem_cap, interval)
    return pack_slots(out["count"], out["status"], out["t_max_used"], out["objective"],
                      out["splits"], n)
