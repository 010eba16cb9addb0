"""Multi-GPU sharding and the stats all-reduce.

Instances are independent, so the only data-path decision is which global
instance ids a rank owns; the only collective is the north_star's
``all_reduce(SUM)`` of the int64[8] statistics vector (accuracy and
deadline-miss counts).  Integer sums make the result identical
for any world size.
"""
from __future__ import annotations


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous strong-scaling shard [floor(w B / W), floor((w+1) B / W))."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return (n_total * rank) // world, (n_total * (rank + 1)) // world


def weak_shard(n_per_rank: int, rank: int) -> tuple[int, int]:
    """Weak scaling: every rank solves its own full batch of distinct global ids."""
    return rank * n_per_rank, (rank + 1) * n_per_rank


def reduce_stats(stats, group=None):
    """all_reduce(SUM) of the int64[8] stats tensor in place (NCCL on GPUs, gloo on CPU)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=group)
    return stats


def derived_metrics(stats) -> dict:
    """Expected accuracy (sum of kept confidence / tasks; drops count 0, reading R15) and the
    planned deadline-miss rate (dropped / tasks) from a reduced stats vector."""
    s = [int(x) for x in stats]
    tasks = max(s[1], 1)
    return {"instances": s[0], "tasks": s[1], "accuracy": s[6] / 1e6 / tasks, "miss_rate": s[2] / tasks,
            "optional_kept_fraction": s[4] / max(s[5], 1), "not_ok_instances": s[3]}


_MIX = 0x9E3779B97F4A7C15 - (1 << 64)  # golden-ratio multiplier as a signed int64


def result_hash(outputs: dict, task_begin, id0: int, n_tasks: int | None = None):
    """int64 fingerprint of a shard's plans (kept, start, finish per task, keyed by global
    instance id), summed modulo 2^64 so that all_reduce(SUM) over any sharding of the same
    global ids yields the same value.  Works on CPU or CUDA tensors."""
    import torch
    kept = outputs["kept"].long()
    start = outputs["start"].long()
    finish = outputs["finish"].long()
    tb = task_begin.long()
    B = tb.numel() - 1
    T = kept.numel()
    dev = kept.device
    inst = torch.repeat_interleave(torch.arange(B, device=dev), tb[1:] - tb[:-1]) if n_tasks is None else \
        torch.arange(T, device=dev) // n_tasks
    local = torch.arange(T, device=dev) - tb[inst]
    v = (kept + 2) * 1000003 + start * 7919 + finish
    gid = inst + id0
    w = (gid * 2 + 1) * _MIX + local * 0x632BE59BD9B4E019  # int64 wraparound arithmetic
    return (v * w).sum()
