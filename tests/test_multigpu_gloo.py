"""World-size-2 gloo test of the multi-GPU plumbing on CPU (no GPU needed).

Each rank takes its shard of global instance ids, produces rank-local results
(the solver has no CPU path, so the oracle stands in for the GPU here, as
SURVEY §4.2 prescribes), builds the stats vector and all-reduces it with the
product's ``reduce_stats``.  The reduced vector must equal the single-process
stats over the whole batch, for strong and weak sharding.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
import oracle
from paper_2011_01112_b200.multigpu import derived_metrics, reduce_stats, result_hash, shard_range, weak_shard
from tests.gpu_util import stats_from

B = 96


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _solve(lo, hi):
    cw = gen.CONFIGS["C2"]
    batch = gen.generate(cw, hi - lo, id_offset=lo)
    out = oracle.solve(batch, oracle.OracleConfig(epsilon_micro=cw.epsilon_micro, max_tasks=32,
                                                  max_horizon=1024), oracle.TIME)
    return batch, out


def _stats_for(lo, hi):
    batch, out = _solve(lo, hi)
    return stats_from(out, batch)


def _hash_for(lo, hi):
    batch, out = _solve(lo, hi)
    t = {k: torch.from_numpy(out[k]) for k in ("kept", "start", "finish")}
    return result_hash(t, torch.from_numpy(batch.task_begin), lo)


def _worker(rank, world, port, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(B, rank, world) if mode == "strong" else weak_shard(B // world, rank)
    st = torch.from_numpy(_stats_for(lo, hi))
    reduce_stats(st)
    h = _hash_for(lo, hi).reshape(1)
    dist.all_reduce(h)
    if rank == 0:
        q.put((st.numpy().tolist(), int(h.item())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["strong", "weak"])
def test_stats_allreduce_world2(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, h = q.get(timeout=240)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    ref = _stats_for(0, B)
    np.testing.assert_array_equal(np.array(got), ref)
    if mode == "strong":  # same global ids, any sharding -> same fingerprint
        assert h == int(_hash_for(0, B).item())
    m = derived_metrics(ref)
    assert 0 < m["accuracy"] <= 1 and 0 <= m["miss_rate"] <= 1


def test_shards_cover_ids_exactly():
    for total in (0, 1, 7, 1 << 24):
        for world in (1, 2, 3, 8):
            spans = [shard_range(total, w, world) for w in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
