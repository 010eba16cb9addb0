"""Helpers that turn hand-written task lists into C-ABI batches (test plumbing)."""
from __future__ import annotations

import numpy as np

from gen import Batch, concat


def batch_from_tasks(tasks, stride: int | None = None) -> Batch:
    """tasks: list of dict(r, d, m, w=[...], a0, g=[...]) -> one-instance Batch."""
    N = len(tasks)
    S = max([len(t["w"]) for t in tasks] + [0])
    st = S if stride is None else stride
    ow = np.zeros((N, st), np.int32)
    og = np.zeros((N, st), np.int32)
    for i, t in enumerate(tasks):
        ow[i, :len(t["w"])] = t["w"]
        og[i, :len(t["g"])] = t["g"]
    return Batch(np.array([0, N], np.int64),
                 np.array([t["r"] for t in tasks], np.int32),
                 np.array([t["d"] for t in tasks], np.int32),
                 np.array([t["m"] for t in tasks], np.int32),
                 np.array([len(t["w"]) for t in tasks], np.uint8), ow,
                 np.array([t["a0"] for t in tasks], np.uint32), og)


def batch_from_many(task_lists, stride: int) -> Batch:
    return concat([batch_from_tasks(t, stride) for t in task_lists], stride)
